"""Per-tile precision gate of the tensor-core E step: E_tile = R_tile·sqrt(1 + max α) of every
64-target tile of the prepared target, and the share of tiles that take the tile-centred residual
(E_tile ≤ gate·σ) along a registration's σ² trace; plus E-step time per residual mode.
python tools/tile_stats.py [configs]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2103_15039_b200 as lsg  # noqa: E402
import synth  # noqa: E402

TILE_BYTES, HDR = 10240, 256


def tile_E(tgt):
    M_pad = (tgt.M + 255) // 256 * 256
    off = HDR + M_pad * 16 * 4
    T = M_pad // 64
    raw = tgt.buf[off: off + T * TILE_BYTES].view(torch.float32).reshape(T, TILE_BYTES // 4).cpu().numpy()
    # core: pair block i (targets 2i, 2i+1) = 16 floats, field f of lane k at 2f + k; meta = field 7
    c = np.stack([raw[:, 14], raw[:, 15], raw[:, 16 + 14]], 1)
    E = raw[:, 16 + 15]
    return E, c


def main():
    cfgs = sys.argv[1:] or ["object", "rgbd", "lidar", "scale"]
    gate = lsg.get_option("tile_gate")
    for name in cfgs:
        wl = synth.make(name)
        tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
        X = torch.from_numpy(wl.source).cuda()
        E, _ = tile_E(tgt)
        real = E > 0
        out = lsg.register(tgt, X, wl.iters, w=wl.w, traces=True)
        tr = out["sigma2_trace"]
        print(f"{name}: M={wl.M} tiles={len(E)}  E_tile pct 50/90/99 = "
              f"{np.percentile(E[real], 50):.3g} / {np.percentile(E[real], 90):.3g} / {np.percentile(E[real], 99):.3g}"
              f"  gate={gate}")
        for k in sorted({0, len(tr) // 4, len(tr) // 2, len(tr) - 1}):
            s = float(np.sqrt(tr[k]))
            print(f"   iter {k:3d} sigma2 {tr[k]:.3e}: centred tiles {np.mean(E[real] <= gate * s):6.1%}")
        run = lsg.EstepRunner(tgt, X)
        for s2 in (float(tr[0]), float(tr[-1])):
            for g in (0.0, gate, 1e30):
                with lsg.options(tile_gate=g):
                    run(out["R"], out["t"], s2, wl.w)
                    torch.cuda.synchronize()
                    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
                    reps = 3 if wl.M > 200000 else 20
                    e0.record()
                    for _ in range(reps):
                        run(out["R"], out["t"], s2, wl.w)
                    e1.record()
                    torch.cuda.synchronize()
                    ms = e0.elapsed_time(e1) / reps
                print(f"   E step sigma2 {s2:.3e} gate {g:8.3g}: {ms:9.3f} ms  {wl.M * wl.N / ms / 1e9:.3e} pairs/s")


if __name__ == "__main__":
    main()
