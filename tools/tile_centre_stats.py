"""Tile meta of prepared targets: R_tile percentiles and the share of tiles whose centre fell back to c_a = 0 on
an axis (y - c not exact in FP32).  Diagnostic.  python tools/tile_centre_stats.py"""
import os, sys, numpy as np, torch
sys.path.insert(0, os.getcwd())
import paper_2103_15039_b200 as lsg, synth
for name in ["object", "lidar"]:
    wl = synth.make(name)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    M_pad = (tgt.M + 255) // 256 * 256
    off = 256 + M_pad * 64
    T = M_pad // 64
    raw = tgt.buf[off: off + T * 10240].view(torch.float32).reshape(T, 2560).cpu().numpy()
    c = np.stack([raw[:, 14], raw[:, 15], raw[:, 30]], 1)
    E = raw[:, 31]; R = raw[:, 46]
    real = E > 0
    print(name, "R pct 50/90", np.percentile(R[real], 50), np.percentile(R[real], 90), "c zero share per axis", (c[real] == 0).mean(0))
