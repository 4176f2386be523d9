"""O2: the paper's matrix form of the E step, Eq. 9-10, in NumPy.  TEST INFRASTRUCTURE ONLY.

    P_mn = K_mn / (Σ_m K_mn + γ),   γ = (2πσ²)^{3/2} / V                         (Eq. 9)
    K    = C ⊙ exp(-(D A + B) / (2σ²))                                          (Eq. 10)
    A_mn = (N R Xᵀ + N t 1ᵀ - s 1ᵀ)_mn²,   s_m = y_mᵀ n_m
    B    = Q + tᵀt 𝟙𝟙ᵀ + 2(1 tᵀ R Xᵀ - Y R Xᵀ - Y t 1ᵀ),  Q_mn = ||x_n||² + ||y_m||²  (reading R2)
    C_mn = (1-w_n)/w_n · π(m)  [· sqrt(1+α_m) in the consistent-normaliser reading R1],  D = diag(α)
Written from the paper's formulas; shares nothing with oracle/lsgcpd_oracle.c.  w > 0 only (Eq. 9
divides by w).  Small M, N only (dense M×N arrays).
"""
from __future__ import annotations

import numpy as np


def correspondence(Y, normals, alpha, X, R, t, sigma2, w, V, consistent=True):
    Y = np.asarray(Y, np.float64)
    Nm = np.asarray(normals, np.float64)
    X = np.asarray(X, np.float64)
    R = np.asarray(R, np.float64)
    t = np.asarray(t, np.float64).reshape(3, 1)
    M, N = Y.shape[0], X.shape[0]
    one_N = np.ones((N, 1))
    one_M = np.ones((M, 1))
    s = np.einsum("mi,mi->m", Y, Nm).reshape(M, 1)
    A = (Nm @ R @ X.T + Nm @ t @ one_N.T - s @ one_N.T) ** 2
    Qm = (X ** 2).sum(axis=1)[None, :] + (Y ** 2).sum(axis=1)[:, None]
    B = Qm + float((t.T @ t)[0, 0]) * np.ones((M, N)) + 2.0 * (one_M @ t.T @ R @ X.T - Y @ R @ X.T - Y @ t @ one_N.T)
    Dg = np.diag(np.asarray(alpha, np.float64))
    C = np.full((M, N), (1.0 - w) / w / M)
    if consistent:
        C = C * np.sqrt(1.0 + np.asarray(alpha, np.float64))[:, None]
    K = C * np.exp(-(Dg @ A + B) / (2.0 * sigma2))
    gamma = (2.0 * np.pi * sigma2) ** 1.5 / V
    denom = K.sum(axis=0, keepdims=True) + gamma
    return K / denom, gamma / denom[0]
