"""Oracle E step (Eq. 5 with Eq. 1-2 densities).  TEST INFRASTRUCTURE ONLY.

The record layout (per source point, 16 numbers) is documented in oracle/lsgcpd_oracle.c and
include/lsgcpd.h; the two are written independently and agree by definition, not by sharing code.
"""
from __future__ import annotations

import numpy as np

from ._lib import f64, lib, ptr

REC = 16
# record column names (same meaning as the product ABI, defined independently)
COLS = ["P", "Py_x", "Py_y", "Py_z", "A_xx", "A_xy", "A_xy_z", "A_yy", "A_yz", "A_zz",
        "b_x", "b_y", "b_z", "D", "lnp", "Pout"]


def estep(Y, normals, alpha, X, R, t, sigma2: float, w: float, V: float, consistent: bool = True,
          nthreads: int = 0) -> np.ndarray:
    """Per-point record (N×16 float64) of the E step at pose (R, t) and σ²."""
    Y, normals, alpha, X = f64(Y), f64(normals), f64(alpha), f64(X)
    R, t = f64(R).reshape(9), f64(t).reshape(3)
    M, N = Y.shape[0], X.shape[0]
    rec = np.empty((N, REC), dtype=np.float64)
    if N == 0:
        return rec
    lib().ora_estep(ptr(Y), ptr(normals), ptr(alpha), M, ptr(X), N, ptr(R), ptr(t), float(sigma2), float(w),
                    float(V), int(bool(consistent)), ptr(rec), int(nthreads))
    return rec


def estep_cf(Y, normals, alpha, prior, X, wn, R, t, sigma2: float, V: float, consistent: bool = True,
             nthreads: int = 0) -> np.ndarray:
    """E-step record with per-component priors π(m) and per-point outlier weights w_n (Eq. 8, P:248-255;
    Eq. 1 and Eq. 5 with π(m), w_n in place of 1/M, w)."""
    Y, normals, alpha, prior, X, wn = f64(Y), f64(normals), f64(alpha), f64(prior), f64(X), f64(wn)
    R, t = f64(R).reshape(9), f64(t).reshape(3)
    M, N = Y.shape[0], X.shape[0]
    if prior.shape != (M,) or wn.shape != (N,):
        raise ValueError("prior must be [M], wn must be [N]")
    rec = np.empty((N, REC), dtype=np.float64)
    if N == 0:
        return rec
    lib().ora_estep_cf(ptr(Y), ptr(normals), ptr(alpha), ptr(prior), M, ptr(X), ptr(wn), N, ptr(R), ptr(t),
                       float(sigma2), float(V), int(bool(consistent)), ptr(rec), int(nthreads))
    return rec


def posterior(Y, normals, alpha, X, R, t, sigma2: float, w: float, V: float, consistent: bool = True):
    """Full posterior matrix P (M×N) and outlier posterior (N,) — small sizes only."""
    Y, normals, alpha, X = f64(Y), f64(normals), f64(alpha), f64(X)
    R, t = f64(R).reshape(9), f64(t).reshape(3)
    M, N = Y.shape[0], X.shape[0]
    P = np.empty((M, N), dtype=np.float64)
    Po = np.empty(N, dtype=np.float64)
    lib().ora_posterior(ptr(Y), ptr(normals), ptr(alpha), M, ptr(X), N, ptr(R), ptr(t), float(sigma2), float(w),
                        float(V), int(bool(consistent)), ptr(P), ptr(Po))
    return P, Po


def sym6(a6: np.ndarray) -> np.ndarray:
    """(…,6) [xx,xy,xz,yy,yz,zz] → (…,3,3) symmetric."""
    a6 = np.asarray(a6)
    out = np.empty(a6.shape[:-1] + (3, 3), dtype=a6.dtype)
    out[..., 0, 0] = a6[..., 0]
    out[..., 0, 1] = out[..., 1, 0] = a6[..., 1]
    out[..., 0, 2] = out[..., 2, 0] = a6[..., 2]
    out[..., 1, 1] = a6[..., 3]
    out[..., 1, 2] = out[..., 2, 1] = a6[..., 4]
    out[..., 2, 2] = a6[..., 5]
    return out
