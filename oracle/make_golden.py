"""Write oracle-only golden files under tests/golden/ (TEST INFRASTRUCTURE ONLY).

Every number written here comes from oracle/ on synth/ inputs; nothing comes from the CUDA path.
    python -m oracle.make_golden object [rgbd lidar rgbd_cf ...]
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

import synth
from oracle import register_workload, se3

OUT = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def make(name: str, iters=None):
    wl = synth.make(name)
    t0 = time.time()
    out = register_workload(wl, iters=iters)
    dt = time.time() - t0
    tr = out["trace"]
    g = {
        "config": name,
        "source": "oracle/make_golden.py (FP64 CPU oracle only); inputs synth.make(%r)" % name,
        "target_sha": digest(wl.target), "source_sha": digest(wl.source),
        "M": wl.M, "N": wl.N, "w": wl.w, "iters": out["iters"], "knn_k": wl.knn_k,
        "V": out["V"], "extent": out["extent"],
        "R": out["R"].tolist(), "t": out["t"].tolist(), "sigma2": out["sigma2"],
        "nll_trace": tr["nll"], "sigma2_trace": tr["sigma2"],
        "R_trace": [r.tolist() for r in tr["R"]], "t_trace": [t.tolist() for t in tr["t"]],
        "rot_err_vs_expected": se3.rotation_angle(out["R"].T @ wl.R_expected),
        "trans_err_vs_expected": float(np.linalg.norm(out["t"] - wl.t_expected)),
        "oracle_seconds": dt, "oracle_e_seconds": tr["e_time"],
    }
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(OUT, f"{name}_oracle.json"), "w") as f:
        json.dump(g, f, indent=1)
    print(name, "done in %.1fs" % dt, "rot err %.2e" % g["rot_err_vs_expected"])


def make_cf(iters: int = 50):
    """The RGBD-CF workload (NEXT-2): depth confidences (reading R23), truncation at φ < 0.04,
    priors π(m) on the truncated target and per-point w_n on the truncated source, whole oracle pipeline."""
    from oracle import outlier as ol
    from oracle import prepare_target, register, working_volume
    wl = synth.make("rgbd")
    thr = np.float32(0.04)
    phi_y = ol.depth_confidence(wl.target[:, 2].astype(np.float64)).astype(np.float32)
    phi_x = ol.depth_confidence(wl.source[:, 2].astype(np.float64)).astype(np.float32)
    Y, py, _ = ol.truncate(wl.target, phi_y, thr)
    X, px, _ = ol.truncate(wl.source, phi_x, thr)
    t0 = time.time()
    tgt = prepare_target(Y, wl.knn_k)
    V, extent = working_volume(Y)
    out = register(tgt, X, wl.w, iters, V, extent, prior=ol.confidence_prior(py.astype(np.float64)),
                   phi_x=px.astype(np.float64))
    dt = time.time() - t0
    tr = out["trace"]
    g = {
        "config": "rgbd_cf",
        "source": "oracle/make_golden.py make_cf (FP64 CPU oracle only); inputs synth.make('rgbd') truncated "
                  "at phi < 0.04 by oracle.outlier.truncate",
        "target_sha": digest(Y), "source_sha": digest(X), "M": int(Y.shape[0]), "N": int(X.shape[0]),
        "w": wl.w, "iters": iters, "knn_k": wl.knn_k, "V": V, "extent": extent,
        "R": out["R"].tolist(), "t": out["t"].tolist(), "sigma2": out["sigma2"],
        "nll_trace": tr["nll"], "sigma2_trace": tr["sigma2"],
        "rot_err_vs_expected": se3.rotation_angle(out["R"].T @ wl.R_expected),
        "trans_err_vs_expected": float(np.linalg.norm(out["t"] - wl.t_expected)),
        "oracle_seconds": dt,
    }
    with open(os.path.join(OUT, "rgbd_cf_oracle.json"), "w") as f:
        json.dump(g, f, indent=1)
    print("rgbd_cf done in %.1fs" % dt, "rot err %.2e" % g["rot_err_vs_expected"])


def make_ext(name: str):
    """object_eta (w from the outlier ratio η = 0.1, Eq. 7) and object_affine (the affine group): the
    object config's whole oracle pipeline with one model extension."""
    from oracle import prepare_target, register, working_volume
    wl = synth.make("object")
    t0 = time.time()
    tgt = prepare_target(wl.target, wl.knn_k)
    V, extent = working_volume(wl.target)
    kw = {"eta": 0.1} if name == "object_eta" else {"group": "affine"}
    out = register(tgt, wl.source, wl.w, wl.iters, V, extent, **kw)
    dt = time.time() - t0
    g = {"config": name, "source": "oracle/make_golden.py make_ext (FP64 CPU oracle only); inputs synth.make('object')",
         "target_sha": digest(wl.target), "source_sha": digest(wl.source), "M": wl.M, "N": wl.N, "w": wl.w,
         "extension": kw, "iters": wl.iters, "V": V, "extent": extent, "R": out["R"].tolist(),
         "t": out["t"].tolist(), "sigma2": out["sigma2"], "sigma2_trace": out["trace"]["sigma2"],
         "oracle_seconds": dt}
    with open(os.path.join(OUT, f"{name}_oracle.json"), "w") as f:
        json.dump(g, f, indent=1)
    print(name, "done in %.1fs" % dt)


if __name__ == "__main__":
    for n in sys.argv[1:]:
        if n == "rgbd_cf":
            make_cf()
        elif n in ("object_eta", "object_affine"):
            make_ext(n)
        else:
            make(n)
