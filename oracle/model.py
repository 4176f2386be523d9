"""Oracle: target-side GMM construction (§3.1).  TEST INFRASTRUCTURE ONLY.

* kNN neighbourhood (k nearest, self included, ties to the lower id) — SPEC S:98-112, S:145;
  neighbourhood type k-NN is reading R9 (the paper does not say).
* surface variation κ = λ_min / (λ1+λ2+λ3) of the neighbourhood covariance, normal = eigenvector
  of λ_min; κ clamped to [1e-12, 1/3], zero trace → degenerate.
* α from the modified logistic sigmoid, Eq. 3, evaluated literally.
* working volume V = AABB of the target inflated by a margin per side (reading R5).
* σ²₀ "similar to CPD": Σ_mn ||x̂_n - y_m||² / (3MN) (reading R7).
"""
from __future__ import annotations

import numpy as np

from ._lib import f64, lib, ptr

KAPPA_FLOOR = 1e-12


def knn(P: np.ndarray, k: int, queries=None, nthreads: int = 0):
    """Exact brute-force kNN (self included; ties → lower id).  Returns (idx int32 [nq,k], d2 float64)."""
    P = f64(P)
    M = P.shape[0]
    if queries is None:
        nq = M
        qptr = None
    else:
        queries = np.ascontiguousarray(queries, dtype=np.int64)
        nq = queries.shape[0]
        qptr = queries.ctypes.data
    idx = np.empty((nq, k), dtype=np.int32)
    d2 = np.empty((nq, k), dtype=np.float64)
    lib().ora_knn(ptr(P), M, qptr, nq, int(k), idx.ctypes.data, d2.ctypes.data, int(nthreads))
    return idx, d2


def alpha_from_kappa(kappa, lam: float = 0.5, alpha_max: float = 50.0):
    """Eq. 3: α = (1 - exp(λ(3 - 1/κ))) / (1 + exp(λ(3 - 1/κ))) · α_max."""
    kappa = np.asarray(kappa, dtype=np.float64)
    e = np.exp(lam * (3.0 - 1.0 / kappa))
    return (1.0 - e) / (1.0 + e) * alpha_max


def local_surface(P: np.ndarray, idx: np.ndarray):
    """Normals and surface variation from neighbour index lists."""
    P = f64(P)
    nb = P[idx]                                    # [M, k, 3]
    c = nb - nb.mean(axis=1, keepdims=True)
    C = np.einsum("mki,mkj->mij", c, c) / idx.shape[1]
    evals, evecs = np.linalg.eigh(C)               # ascending eigenvalues (LAPACK)
    trace = evals.sum(axis=1)
    degenerate = ~(trace > 0.0)
    kappa = np.where(degenerate, 1.0 / 3.0, evals[:, 0] / np.where(degenerate, 1.0, trace))
    kappa = np.clip(kappa, KAPPA_FLOOR, 1.0 / 3.0)
    normals = evecs[:, :, 0].copy()
    normals[degenerate] = np.array([0.0, 0.0, 1.0])
    return normals, kappa, degenerate, evals


def prepare_target(Y: np.ndarray, k: int = 10, alpha_max: float = 50.0, lam: float = 0.5,
                   nthreads: int = 0, idx=None):
    """Annotate the target: kNN → κ, n → α (Eq. 3).  Returns a dict of float64 arrays."""
    Y = f64(Y)
    if idx is None:
        idx, _ = knn(Y, k, nthreads=nthreads)
    normals, kappa, degenerate, evals = local_surface(Y, idx)
    alpha = alpha_from_kappa(kappa, lam, alpha_max)
    return {"Y": Y, "normals": normals, "kappa": kappa, "alpha": alpha, "degenerate": degenerate,
            "knn": idx, "evals": evals}


def mean_nn_spacing(Y: np.ndarray, nthreads: int = 0) -> float:
    """Mean distance to the nearest OTHER point (used only for a zero-extent axis)."""
    idx, d2 = knn(Y, 2, nthreads=nthreads)
    self_id = np.arange(Y.shape[0])
    d_other = np.where(idx[:, 0] == self_id, d2[:, 1], d2[:, 0])
    return float(np.sqrt(d_other).mean())


def working_volume(Y: np.ndarray, margin: float = 0.1, nthreads: int = 0):
    """V = Π_a extent_a (1 + 2·margin); a zero-extent axis is floored at the mean NN spacing.
    Returns (V, extent) with extent = diagonal of the (un-inflated) AABB."""
    Y = f64(Y)
    ext = Y.max(axis=0) - Y.min(axis=0)
    extent = float(np.sqrt((ext ** 2).sum()))
    if np.any(ext <= 0.0):
        s = mean_nn_spacing(Y, nthreads)
        ext = np.where(ext <= 0.0, s, ext)
    V = float(np.prod(ext * (1.0 + 2.0 * margin)))
    return V, extent


def sigma2_init(X: np.ndarray, Y: np.ndarray, R=None, t=None) -> float:
    """σ²₀ = Σ_{m,n} ||x̂_n - y_m||² / (3MN) in the exact centred closed form
    M Σ_n ||x̂_n - ȳ||² + N Σ_m ||y_m - ȳ||²   (the cross term vanishes since Σ_m (y_m - ȳ) = 0)."""
    X = f64(X)
    Y = f64(Y)
    if R is not None:
        X = X @ np.asarray(R, dtype=np.float64).T + np.asarray(t, dtype=np.float64)
    M, N = Y.shape[0], X.shape[0]
    yb = Y.mean(axis=0)
    sx = ((X - yb) ** 2).sum()
    sy = ((Y - yb) ** 2).sum()
    return float((M * sx + N * sy) / (3.0 * M * N))


def sum_sq_pairs(X: np.ndarray, Y: np.ndarray, nthreads: int = 0) -> float:
    """Σ_{m,n} ||x_n - y_m||² by the plain double loop (C)."""
    X = f64(X)
    Y = f64(Y)
    return float(lib().ora_sum_sq_pairs(ptr(X), X.shape[0], ptr(Y), Y.shape[0], int(nthreads)))
