"""One lsgcpd_estep launch on a BASELINE config (for ncu captures).  VARIANT env selects the kernel."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_2103_15039_b200 as lsg
cfg = os.environ.get("CFG", "scale")
os.environ["LSGCPD_ESTEP_VARIANT"] = os.environ.get("VARIANT", "0")
wl = synth.make(cfg)
rng = np.random.default_rng(0)
n = rng.standard_normal(wl.target.shape); n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
a = rng.uniform(0, 50, wl.M).astype(np.float32)
tgt = lsg.pack_target(torch.from_numpy(wl.target).cuda(), torch.from_numpy(n).cuda(), torch.from_numpy(a).cuda())
run = lsg.EstepRunner(tgt, torch.from_numpy(wl.source).cuda())
for _ in range(int(os.environ.get("REPS", "2"))):
    run(wl.R_expected, wl.t_expected, 1e-3, float(os.environ.get("W", wl.w)))
torch.cuda.synchronize()
print("ok", float(run.rec[:, 0].sum()))
