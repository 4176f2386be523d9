"""Parity helpers shared by the -m gpu tests (tolerances: DESIGN.md "Parity protocol")."""
import numpy as np

TOL = 2e-5          # north star: per-point statistics within relative 2e-5 (FP32)
P_FLOOR = 1e-6      # inlier-mass floor of the scale (points with negligible mass)


def record_errors(gpu: np.ndarray, ora: np.ndarray, Y: np.ndarray, alpha: np.ndarray):
    """Scaled element-wise errors |gpu - ora| / scale for every record component."""
    gpu = np.asarray(gpu, np.float64)
    ora = np.asarray(ora, np.float64)
    ymax = float(np.abs(Y).max())
    amax = max(float(np.max(alpha)), 1.0)
    sP = np.maximum(ora[:, 0], P_FLOOR)
    scale = np.empty_like(ora)
    scale[:, 0] = sP
    scale[:, 1:4] = (sP * ymax)[:, None]
    scale[:, 4:10] = (sP * amax)[:, None]
    scale[:, 10:13] = (sP * amax * ymax)[:, None]
    scale[:, 13] = np.maximum(ora[:, 13], P_FLOOR)
    scale[:, 14] = np.maximum(np.abs(ora[:, 14]), 1.0)
    scale[:, 15] = np.maximum(ora[:, 15], P_FLOOR)
    return np.abs(gpu - ora) / scale


def assert_record_parity(gpu, ora, Y, alpha, tol=TOL, what=""):
    err = record_errors(gpu, ora, Y, alpha)
    worst = err.max(axis=0)
    n_floor = int((np.asarray(ora)[:, 0] < P_FLOOR).sum())
    msg = f"{what}: max scaled error per column {np.array2string(worst, precision=2)}; " \
          f"p99 {np.percentile(err, 99):.2e}; floor-limited points {n_floor}"
    assert np.all(np.isfinite(np.asarray(gpu))), what + ": non-finite GPU record"
    assert worst.max() <= tol, msg
    return err
