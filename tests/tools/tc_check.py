"""Quick check of the tensor-core E step: parity vs the oracle (tiny, sampled scale) and speed vs CUDA-core."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth, oracle
import paper_2103_15039_b200 as lsg
from tests.parity import record_errors
for cfg in os.environ.get("CFGS", "tiny,scale").split(","):
    wl = synth.make(cfg)
    rng = np.random.default_rng(0)
    n = rng.standard_normal(wl.target.shape); n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    a = rng.uniform(0, 50, wl.M).astype(np.float32)
    tgt = lsg.pack_target(torch.from_numpy(wl.target).cuda(), torch.from_numpy(n).cuda(), torch.from_numpy(a).cuda())
    X = torch.from_numpy(wl.source).cuda()
    idx = np.arange(wl.N) if wl.N <= 2000 else np.sort(rng.choice(wl.N, 64, replace=False))
    for s2 in (oracle.sigma2_init(wl.source, wl.target, wl.R_expected, wl.t_expected), 1e-3, 1e-5):
        ora = oracle.estep(wl.target, n.astype(np.float64), a.astype(np.float64), wl.source[idx], wl.R_expected, wl.t_expected, s2, wl.w, tgt.volume)
        for tc in os.environ.get("TCS", "1:0,0").split(","):
            on, _, tv = tc.partition(":")
            os.environ["LSGCPD_TC"] = on
            os.environ["LSGCPD_TC_VARIANT"] = tv or "0"
            run = lsg.EstepRunner(tgt, X)
            run(wl.R_expected, wl.t_expected, s2, wl.w); torch.cuda.synchronize()
            err = record_errors(run.rec.cpu().numpy()[idx], ora, wl.target, a)
            reps = 2 if cfg == "scale" else 20
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                run(wl.R_expected, wl.t_expected, s2, wl.w)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            print(f"{cfg} s2={s2:.1e} tc={tc}: {ms:9.3f} ms {wl.M*wl.N/ms/1e9:.3e} pairs/s  err max {err.max():.1e} per-col {np.array2string(err.max(0), precision=0)}", flush=True)
