"""Max scaled E-step error vs the oracle per tile-gate value (DESIGN §8 "tile-centred residual"), without and with
the far-point rule: object and rgbd (full records), tiny, lidar and scale (4,096 sampled points), at σ²₀, 1e-3,
1e-4 and the converged σ² of the goldens.  Diagnostic (imports the oracle).
python tests/tools/gate_sweep.py [config ...]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import paper_2103_15039_b200 as lsg  # noqa: E402
from tests.gpu_common import oracle_target32  # noqa: E402
from tests.parity import record_errors, transformed  # noqa: E402

SWEEPS = [("G", "tile_gate", [0.0, 8.0, 16.0, 24.0, 32.0, 48.0, 1e30], {"far_rule": 0}),
          ("G+far", "tile_gate", [0.0, 24.0, 48.0], {"far_rule": 1})]
for name in sys.argv[1:] or ["tiny", "object", "rgbd", "lidar", "scale"]:
    wl, n32, a32, V, ext = oracle_target32(name)
    tgt = lsg.pack_target(torch.from_numpy(wl.target).cuda(), torch.from_numpy(n32).cuda(), torch.from_numpy(a32).cuda())
    X = torch.from_numpy(wl.source).cuda()
    R, t = wl.R_expected, wl.t_expected
    idx = np.sort(np.random.default_rng(5).choice(wl.N, 4096, replace=False)) if wl.N > 200_000 else np.arange(wl.N)
    s2s = [oracle.sigma2_init(wl.source, wl.target, R, t), 1e-3, 1e-4]
    gp = os.path.join(ROOT, "tests", "golden", f"{name}_oracle.json")
    if os.path.exists(gp):
        s2s.append(float(json.load(open(gp))["sigma2"]))
    if name == "scale":
        s2s = [s2s[0], 2.06e-2, 1e-3]   # σ²₀, the converged σ² of the bench registration, 1e-3
    Xh = transformed(wl.source[idx], R, t)
    for s2 in s2s:
        ora = oracle.estep(wl.target, n32.astype(np.float64), a32.astype(np.float64), wl.source[idx], R, t, s2,
                           wl.w, V)
        for label, opt, values, fixed in SWEEPS:
            row = []
            for g in values:
                with lsg.options(tc=1, **{opt: g}, **fixed):
                    rec = lsg.estep(tgt, X, R, t, s2, wl.w, V).cpu().numpy()[idx]
                row.append(record_errors(rec, ora, wl.target, a32, Xh, s2).max())
            print(f"{name:7s} s2={s2:.3e} " + " ".join(f"{label}={g:g}:{e:.2e}" for g, e in zip(values, row)),
                  flush=True)
