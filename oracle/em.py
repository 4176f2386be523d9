"""Oracle EM loop (§3.1 E/M steps).  TEST INFRASTRUCTURE ONLY.

for k in 0..iters-1:  E step at (g_k, σ²_k) → record (NLL_k = -Σ_n ln p(x̂_n), Eq. 4)
                      M step → (g_{k+1}, σ²_{k+1}).
Fixed iteration count (no early stop, reading R16); initial pose identity unless given (R17);
σ²₀ by the CPD formula (R7); ΣP ≤ 1e-12·N for 3 consecutive iterations aborts ("no mass").
Optional model extensions: eta → w_0 = w_max(η) of §3.2 re-evaluated from σ²_k at every E step (R22);
prior π(m) and phi_x → w_n = 1 - (1 - w_0) φ(x_n) of the confidence filtering, Eq. 8.
"""
from __future__ import annotations

import time

import numpy as np

from .estep import estep, estep_cf
from .model import prepare_target, sigma2_init, working_volume
from .mstep import mstep
from .outlier import outlier_weight_max, point_outlier_weights


def register(target: dict, X, w: float, iters: int, V: float, extent: float, R0=None, t0=None,
             sigma2_0=None, consistent: bool = True, newton_max: int = 10, sigma2_floor_rel: float = 1e-12,
             nthreads: int = 0, keep_records: bool = False, eta=None, prior=None, phi_x=None, group: str = "se3"):
    Y, normals, alpha = target["Y"], target["normals"], target["alpha"]
    general = eta is not None or prior is not None or phi_x is not None
    M = Y.shape[0]
    pi = np.full(M, 1.0 / M) if prior is None else np.asarray(prior, dtype=np.float64)
    X = np.ascontiguousarray(X, dtype=np.float64)
    R = np.eye(3) if R0 is None else np.asarray(R0, dtype=np.float64).copy()
    t = np.zeros(3) if t0 is None else np.asarray(t0, dtype=np.float64).copy()
    s2 = sigma2_init(X, Y, R, t) if sigma2_0 is None or sigma2_0 <= 0 else float(sigma2_0)
    floor = sigma2_floor_rel * extent * extent
    trace = {"nll": [], "sigma2": [s2], "R": [R.copy()], "t": [t.copy()], "sumP": [], "newton": [],
             "records": [], "w0": [], "e_time": 0.0, "m_time": 0.0}
    no_mass = 0
    status = 0
    k_done = 0
    for k in range(iters):
        t0_ = time.perf_counter()
        w0 = outlier_weight_max(eta, V, pi, alpha, s2, consistent) if eta is not None else w
        trace["w0"].append(w0)
        if general:
            wn = point_outlier_weights(w0, phi_x) if phi_x is not None else np.full(X.shape[0], w0)
            rec = estep_cf(Y, normals, alpha, pi, X, wn, R, t, s2, V, consistent, nthreads)
        else:
            rec = estep(Y, normals, alpha, X, R, t, s2, w, V, consistent, nthreads)
        t1_ = time.perf_counter()
        trace["nll"].append(float(-rec[:, 14].sum()))
        if keep_records:
            trace["records"].append(rec)
        R, t, s2, info = mstep(X, rec, R, t, s2, extent, newton_max, floor, group)
        trace["m_time"] += time.perf_counter() - t1_
        trace["e_time"] += t1_ - t0_
        trace["sigma2"].append(s2)
        trace["R"].append(R.copy())
        trace["t"].append(t.copy())
        trace["sumP"].append(info["sumP"])
        trace["newton"].append(info["newton_iters"])
        k_done = k + 1
        no_mass = no_mass + 1 if info["sumP"] <= 1e-12 * X.shape[0] else 0
        if no_mass >= 3:
            status = -5
            break
    return {"R": R, "t": t, "sigma2": s2, "iters": k_done, "status": status, "trace": trace}


def register_workload(wl, iters=None, nthreads: int = 0, keep_records: bool = False, consistent: bool = True,
                      alpha_max: float = 50.0, lam: float = 0.5):
    """Full oracle pipeline on a synth.Workload: prepare → V → σ²₀ → EM."""
    tgt = prepare_target(wl.target, wl.knn_k, alpha_max, lam, nthreads)
    V, extent = working_volume(wl.target, 0.1, nthreads)
    out = register(tgt, wl.source, wl.w, wl.iters if iters is None else iters, V, extent,
                   consistent=consistent, nthreads=nthreads, keep_records=keep_records)
    out["V"], out["extent"], out["target"] = V, extent, tgt
    return out
