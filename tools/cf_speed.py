"""Confidence filtering (NEXT-2) on the RGBD config, all on the GPU: the plain registration of the
full clouds vs the CF pipeline (depth confidences → truncation at φ < 0.04 → target priors π(m) and source
weights w_n → registration), whole-call times including prepare, 50 EM iterations each."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2103_15039_b200 as lsg


def rotation_angle(R):
    """Angle of a rotation matrix (rad)."""
    return float(np.arccos(np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0)))


wl = synth.make("rgbd")
Yd, Xd = torch.from_numpy(wl.target).cuda(), torch.from_numpy(wl.source).cuda()


def plain():
    tgt = lsg.prepare_target(Yd, wl.knn_k)
    return lsg.register(tgt, Xd, wl.iters, w=wl.w), wl.M, wl.N


def cf():
    py, px = lsg.depth_confidence(Yd), lsg.depth_confidence(Xd)
    Y, pyk = lsg.select_confident(Yd, py, 0.04)
    X, pxk = lsg.select_confident(Xd, px, 0.04)
    tgt = lsg.prepare_target(Y, wl.knn_k)
    lsg.set_prior(tgt, pyk)
    return lsg.register(tgt, X, wl.iters, w=wl.w, src_conf=pxk), Y.shape[0], X.shape[0]


for name, fn in (("plain", plain), ("CF", cf)):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(3):
        out, M, N = fn()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 3
    rot = np.degrees(rotation_angle(out["R"].T @ wl.R_expected))
    print(f"{name:5s} M={M:6d} N={N:6d}: {dt * 1e3:7.1f} ms per registration ({1 / dt:5.1f} /s), "
          f"rotation error vs ground truth {rot:.3f} deg, |t - t_gt| {np.linalg.norm(out['t'] - wl.t_expected):.4f}",
          flush=True)
