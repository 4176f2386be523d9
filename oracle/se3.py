"""Oracle SE(3) machinery (§3.5).  TEST INFRASTRUCTURE ONLY.

Basis order (reading R14/S:356): E1..E3 rotations about x, y, z; E4..E6 translations x, y, z.
"""
from __future__ import annotations

import numpy as np


def skew(w) -> np.ndarray:
    w = np.asarray(w, dtype=np.float64)
    return np.array([[0.0, -w[2], w[1]], [w[2], 0.0, -w[0]], [-w[1], w[0], 0.0]])


def basis(i: int) -> np.ndarray:
    """4×4 se(3) basis matrix E_i, i = 1..6."""
    E = np.zeros((4, 4))
    if 1 <= i <= 3:
        e = np.zeros(3)
        e[i - 1] = 1.0
        E[:3, :3] = skew(e)
    elif 4 <= i <= 6:
        E[i - 4, 3] = 1.0
    else:
        raise IndexError(i)
    return E


def hat(xi) -> np.ndarray:
    """ξ = (ω, v) ↦ Σ ξ_i E_i (4×4)."""
    xi = np.asarray(xi, dtype=np.float64)
    out = np.zeros((4, 4))
    out[:3, :3] = skew(xi[:3])
    out[:3, 3] = xi[3:]
    return out


def exp(xi):
    """Closed-form exponential (Rodrigues rotation and V matrix); series below θ = 1e-4."""
    xi = np.asarray(xi, dtype=np.float64)
    w, v = xi[:3], xi[3:]
    th2 = float(w @ w)
    th = np.sqrt(th2)
    K = skew(w)
    K2 = K @ K
    if th < 1e-4:
        # Taylor series of sinθ/θ, (1-cosθ)/θ², (θ-sinθ)/θ³ to O(θ⁶)
        a = 1.0 - th2 / 6.0 + th2 * th2 / 120.0
        b = 0.5 - th2 / 24.0 + th2 * th2 / 720.0
        c = 1.0 / 6.0 - th2 / 120.0 + th2 * th2 / 5040.0
    else:
        a = np.sin(th) / th
        b = (1.0 - np.cos(th)) / th2
        c = (th - np.sin(th)) / (th2 * th)
    R = np.eye(3) + a * K + b * K2
    V = np.eye(3) + b * K + c * K2
    return R, V @ v


def compose(R, t, dR, dt):
    """g ∘ δ for g = (R, t), δ = (dR, dt):  x ↦ R (dR x + dt) + t."""
    return R @ dR, R @ dt + t


def inverse(R, t):
    return R.T, -(R.T @ t)


def homogeneous(R, t) -> np.ndarray:
    g = np.eye(4)
    g[:3, :3] = R
    g[:3, 3] = t
    return g


def rotation_angle(R) -> float:
    """Angle of a rotation matrix (axis-angle magnitude), robust near 0 and π."""
    c = (np.trace(R) - 1.0) / 2.0
    s = np.linalg.norm(np.array([R[2, 1] - R[1, 2], R[0, 2] - R[2, 0], R[1, 0] - R[0, 1]])) / 2.0
    return float(np.arctan2(s, np.clip(c, -1.0, 1.0)))
