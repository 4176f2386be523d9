"""Time lsgcpd_estep on one config for a list of tensor-core variants (no parity; see tests/tools/tc_check.py)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2103_15039_b200 as lsg
cfg = os.environ.get("CFG", "scale"); s2 = float(os.environ.get("S2", "1e-3"))
wl = synth.make(cfg)
rng = np.random.default_rng(0)
n = rng.standard_normal(wl.target.shape); n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
a = rng.uniform(0, 50, wl.M).astype(np.float32)
tgt = lsg.pack_target(torch.from_numpy(wl.target).cuda(), torch.from_numpy(n).cuda(), torch.from_numpy(a).cuda())
X = torch.from_numpy(wl.source).cuda()
for tv in os.environ.get("TCS", "9").split(","):
    os.environ["LSGCPD_TC"] = "1"; os.environ["LSGCPD_TC_VARIANT"] = tv
    run = lsg.EstepRunner(tgt, X)
    run(wl.R_expected, wl.t_expected, s2, wl.w); torch.cuda.synchronize()
    reps = int(os.environ.get("REPS", "3"))
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        run(wl.R_expected, wl.t_expected, s2, wl.w)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"{os.environ.get('TAG', '')} {cfg} tc={tv}: {ms:9.3f} ms  {wl.M * wl.N / ms * 1e3:.4e} pairs/s", flush=True)
