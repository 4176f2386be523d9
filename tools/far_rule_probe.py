"""Potential of the far-point rule when source points are in a spatially coherent (Morton) order: registration
time per EM iteration with the source as given and Morton-sorted, far rule off and on.  Diagnostic.
python tools/far_rule_probe.py [configs]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402


def morton_order(X):
    lo, hi = X.min(0), X.max(0)
    q = np.floor((X - lo) / max(float((hi - lo).max()), 1e-30) * 2097151.0).astype(np.uint64)
    key = np.zeros(len(X), np.uint64)
    for b in range(21):
        for a in range(3):
            key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return np.argsort(key, kind="stable")


for cfg in sys.argv[1:] or ["object", "rgbd", "lidar"]:
    wl = synth.make(cfg)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    for order in ("given", "morton"):
        S = wl.source if order == "given" else wl.source[morton_order(wl.source)]
        X = torch.from_numpy(np.ascontiguousarray(S)).cuda()
        for fr in (0, 1):
            with lsg.options(far_rule=fr):
                reg = lsg.Registrar(tgt, X, wl.iters)
                out = reg(w=wl.w)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                reps = 10 if wl.M < 20000 else 2
                e0.record()
                for _ in range(reps):
                    out = reg(w=wl.w)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / reps
            print(f"{cfg:7s} source {order:6s} far_rule={fr}: {ms / wl.iters * 1e3:9.1f} us/iter  sigma2 {out['sigma2']:.6e}",
                  flush=True)
