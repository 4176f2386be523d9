"""Full-size registrations (GPU-prepared target) vs the FP64 oracle goldens in tests/golden/: how close."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2103_15039_b200 as lsg


def rotation_angle(R):
    """Axis-angle magnitude of a rotation matrix (rad), robust near 0 (atan2 of the skew part and the trace)."""
    s = np.linalg.norm([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]]) / 2.0
    return float(np.arctan2(s, np.clip((np.trace(R) - 1.0) / 2.0, -1.0, 1.0)))

G = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
for name in ("object", "rgbd", "lidar"):
    g = json.load(open(os.path.join(G, f"{name}_oracle.json")))
    wl = synth.make(name)
    tgt = lsg.prepare_target(torch.from_numpy(wl.target).cuda(), wl.knn_k)
    out = lsg.register(tgt, torch.from_numpy(wl.source).cuda(), g["iters"], w=wl.w, traces=True)
    ang = rotation_angle(out["R"].T @ np.array(g["R"]))
    dt = np.linalg.norm(out["t"] - np.array(g["t"])) / g["extent"]
    s2 = abs(out["sigma2"] / g["sigma2"] - 1)
    s2t = np.max(np.abs(np.array(out["sigma2_trace"]) / np.array(g["sigma2_trace"]) - 1))
    print(f"{name:7s} iters={g['iters']:3d}  rot diff {ang:.2e} rad  |dt|/extent {dt:.2e}  sigma2 rel {s2:.2e}"
          f"  max sigma2-trace rel {s2t:.2e}  (oracle {g['oracle_seconds']:.0f} s on its host)", flush=True)

# the RGBD-CF pipeline (NEXT-2): truncation, priors, per-point w_n (the truncation decision repeated here in FP32)
g = json.load(open(os.path.join(G, "rgbd_cf_oracle.json")))
wl = synth.make("rgbd")
thr = np.float32(0.04)


def depth_phi(z, c1=0.002, zmin=0.4):
    return np.clip((c1 * zmin * zmin) / (c1 * z.astype(np.float64) ** 2), 0.0, 1.0).astype(np.float32)


py_all, px_all = depth_phi(wl.target[:, 2]), depth_phi(wl.source[:, 2])
ky, kx = py_all >= thr, px_all >= thr
Y, py, X, px = wl.target[ky], py_all[ky], wl.source[kx], px_all[kx]
tgt = lsg.prepare_target(torch.from_numpy(np.ascontiguousarray(Y)).cuda(), wl.knn_k)
lsg.set_prior(tgt, torch.from_numpy(py).cuda())
out = lsg.register(tgt, torch.from_numpy(np.ascontiguousarray(X)).cuda(), g["iters"], w=wl.w,
                   src_conf=torch.from_numpy(px).cuda(), traces=True)
ang = rotation_angle(out["R"].T @ np.array(g["R"]))
dt = np.linalg.norm(out["t"] - np.array(g["t"])) / g["extent"]
print(f"rgbd_cf iters={g['iters']:3d}  rot diff {ang:.2e} rad  |dt|/extent {dt:.2e}  sigma2 rel "
      f"{abs(out['sigma2'] / g['sigma2'] - 1):.2e}  (M={Y.shape[0]} N={X.shape[0]}; oracle {g['oracle_seconds']:.0f} s)",
      flush=True)
