"""Tile residual modes of the batched problems (NEXT-3): E_tile/σ at the converged σ² of a few desk problems,
and the share of tiles under the centred-residual gate.  python tools/batch_tile_stats.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402
from tools.tile_stats import tile_E  # noqa: E402

gate = lsg.get_option("tile_gate")
for w in synth.make_batch(8, 3500):
    tgt = lsg.prepare_target(torch.from_numpy(w.target).cuda(), w.knn_k)
    out = lsg.register(tgt, torch.from_numpy(w.source).cuda(), w.iters, w=w.w, traces=True)
    E, _ = tile_E(tgt)
    E = E[E > 0]
    tr = out["sigma2_trace"]
    for k in (0, len(tr) // 2, len(tr) - 1):
        s = float(np.sqrt(tr[k]))
        print(f"M={w.M} iter {k:2d} sigma {s:.4f}: E/sigma p50 {np.median(E) / s:7.1f}  centred tiles "
              f"{np.mean(E <= gate * s):6.1%}")
