"""Time lsgcpd_estep per kernel variant (LSGCPD_ESTEP_VARIANT) on BASELINE configs; check sampled parity."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth, oracle
import paper_2103_15039_b200 as lsg
from tests.parity import record_errors

variants = [int(v) for v in os.environ.get("VARIANTS", "0,1,2,3,4,5").split(",")]
configs = os.environ.get("CONFIGS", "scale,object").split(",")
out = {}
for cfg in configs:
    wl = synth.make(cfg)
    rng = np.random.default_rng(0)
    n = rng.standard_normal(wl.target.shape); n = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    a = rng.uniform(0, 50, wl.M).astype(np.float32)
    tgt = lsg.pack_target(torch.from_numpy(wl.target).cuda(), torch.from_numpy(n).cuda(), torch.from_numpy(a).cuda())
    X = torch.from_numpy(wl.source).cuda()
    idx = np.sort(rng.choice(wl.N, 64, replace=False))
    V = tgt.volume
    for s2, w in ((1e-3, wl.w), (1e-3, 0.0)):
        ora = oracle.estep(wl.target, n.astype(np.float64), a.astype(np.float64), wl.source[idx], wl.R_expected, wl.t_expected, s2, w, V)
        for v in variants:
            os.environ["LSGCPD_ESTEP_VARIANT"] = str(v)
            run = lsg.EstepRunner(tgt, X)
            run(wl.R_expected, wl.t_expected, s2, w); torch.cuda.synchronize()
            err = record_errors(run.rec.cpu().numpy()[idx], ora, wl.target, a).max()
            reps = 3 if cfg == "scale" else 50
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(reps):
                run(wl.R_expected, wl.t_expected, s2, w)
            e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            rate = wl.M * wl.N / (ms * 1e-3)
            key = f"{cfg}/w={w}/v{v}"
            out[key] = {"ms": ms, "pairs_per_s": rate, "max_scaled_err": float(err)}
            print(f"{key:24s} {ms:9.3f} ms  {rate:.3e} pairs/s  mufu {rate/4.654e12:.3f}  err {err:.1e}", flush=True)
json.dump(out, open("gpurun_out/estep_speed.json", "w"), indent=1)
