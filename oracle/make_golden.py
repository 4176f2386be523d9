"""Write oracle-only golden files under tests/golden/ (TEST INFRASTRUCTURE ONLY).

Every number written here comes from oracle/ on synth/ inputs; nothing comes from the CUDA path.
    python -m oracle.make_golden object [rgbd lidar ...]
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


if __name__ == "__main__":
    for n in sys.argv[1:]:
        make(n)
