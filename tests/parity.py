"""Parity helpers shared by the -m gpu tests (tolerances: DESIGN.md "Parity protocol").

The north star's "per-point statistics within relative 2e-5" is read per record component as
|gpu - ora| ≤ 2e-5 · scale_c,n, where scale is the component's natural magnitude for point n:
  P, P_out, D       max(value, 1e-6)                      (1e-6: the inlier-mass floor)
  A = Σ P α n nᵀ     max(P, 1e-6) · α_max
  Σ P y             Y_n = Σ_m P_mn ||y_m||, bounded from the oracle's own record (Cauchy-Schwarz, d ≥ ||r||²/σ²):
                    Σ P ||y|| ≤ P ||x̂|| + Σ P ||r|| ≤ P ||x̂|| + sqrt(P · σ² D), floored at 1e-6 · max||y||
  b = Σ P α (n·y) n  α_max · that bound
  ln p              max(|ln p|, 1)
When x̂ and σ² are not given, the y-scale falls back to max(P, 1e-6) · max||y|| (cloud-wide, looser for points
near the origin of a large cloud)."""
import numpy as np

TOL = 2e-5          # north star: per-point statistics within relative 2e-5 (FP32)
P_FLOOR = 1e-6      # inlier-mass floor of the scale (points with negligible mass)


def record_errors(gpu: np.ndarray, ora: np.ndarray, Y: np.ndarray, alpha: np.ndarray, Xh=None, s2=None):
    """Scaled element-wise errors |gpu - ora| / scale for every record component."""
    gpu = np.asarray(gpu, np.float64)
    ora = np.asarray(ora, np.float64)
    ymax = float(np.abs(Y).max())
    amax = max(float(np.max(alpha)), 1.0)
    sP = np.maximum(ora[:, 0], P_FLOOR)
    if Xh is not None and s2 is not None:
        P, D = np.maximum(ora[:, 0], 0.0), np.maximum(ora[:, 13], 0.0)
        ybound = P * np.linalg.norm(np.asarray(Xh, np.float64), axis=1) + np.sqrt(P * float(s2) * D)
        sY = np.maximum(ybound, P_FLOOR * ymax)
    else:
        sY = sP * ymax
    scale = np.empty_like(ora)
    scale[:, 0] = sP
    scale[:, 1:4] = sY[:, None]
    scale[:, 4:10] = (sP * amax)[:, None]
    scale[:, 10:13] = (sY * amax)[:, None]
    scale[:, 13] = np.maximum(ora[:, 13], P_FLOOR)
    scale[:, 14] = np.maximum(np.abs(ora[:, 14]), 1.0)
    scale[:, 15] = np.maximum(ora[:, 15], P_FLOOR)
    return np.abs(gpu - ora) / scale


def transformed(X, R, t):
    """x̂ = R x + t in FP64 (for the local y-scale)."""
    return np.asarray(X, np.float64) @ np.asarray(R, np.float64).T + np.asarray(t, np.float64)


def assert_record_parity(gpu, ora, Y, alpha, tol=TOL, what="", Xh=None, s2=None):
    err = record_errors(gpu, ora, Y, alpha, Xh, s2)
    worst = err.max(axis=0)
    n_floor = int((np.asarray(ora)[:, 0] < P_FLOOR).sum())
    msg = f"{what}: max scaled error per column {np.array2string(worst, precision=2)}; " \
          f"p99 {np.percentile(err, 99):.2e}; floor-limited points {n_floor}"
    assert np.all(np.isfinite(np.asarray(gpu))), what + ": non-finite GPU record"
    assert worst.max() <= tol, msg
    return err
