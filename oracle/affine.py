"""Oracle M step on the affine group (§3.5: "this method can be easily extended to other
types of registration of which the transformation can be represented by a matrix Lie group, e.g., affine
transformation, by replacing the basis matrices in Lie algebra").  TEST INFRASTRUCTURE ONLY.

Group: GA⁺(3), g̃ = [[A, t], [0, 1]] with det A > 0.  Lie algebra aff(3) basis (reading R24), 12 matrices:
E_{3i+j+1} = e_i e_jᵀ in the linear block (i, j = 0..2, row-major), E_{10..12} = translations x, y, z.
With P frozen the objective is the same per-point form as the rigid case (oracle/mstep.py):
    q(g) = Σ_n σ² D_n + 2 Δ_nᵀ u_n + Δ_nᵀ H_n Δ_n,   Δ_n = g(x_n) - x̂_n.
Right derivatives (Eq. 11-12 with the aff(3) basis), of ½q at g ∘ exp(ξ^), ξ = 0, with
z_n = g(x_n), v_n = H_n z_n - g_n (record sums), J_nk = (g̃ E_k x̃_n)[0:3]:
    ∇_k   = Σ_n v_nᵀ J_nk
    H_kl  = Σ_n J_nkᵀ H_n J_nl + v_nᵀ (g̃ ½(E_k E_l + E_l E_k) x̃_n)[0:3]      (symmetrised Eq. 12)
Newton update g ← g ∘ exp(δ^), δ = -(H + μI)⁻¹∇ with the same damping rules as the rigid oracle (R11-R13);
exp is the matrix exponential (scipy.linalg.expm, a library primitive).
"""
from __future__ import annotations

import numpy as np
from scipy.linalg import expm

K_AFF = 12


def basis(k: int) -> np.ndarray:
    """4×4 aff(3) basis matrix E_k, k = 1..12."""
    E = np.zeros((4, 4))
    if 1 <= k <= 9:
        E[(k - 1) // 3, (k - 1) % 3] = 1.0
    elif 10 <= k <= 12:
        E[k - 10, 3] = 1.0
    else:
        raise IndexError(k)
    return E


def hat(xi) -> np.ndarray:
    out = np.zeros((4, 4))
    for k in range(K_AFF):
        out += xi[k] * basis(k + 1)
    return out


def exp(xi):
    """(A, t) of exp(ξ^) (matrix exponential of the 4×4 algebra element)."""
    G = expm(hat(np.asarray(xi, dtype=np.float64)))
    return G[:3, :3], G[:3, 3]


def compose(A, t, dA, dt):
    return A @ dA, A @ dt + t


def grad_hess(stats, A, t):
    """∇ and H of ½q(g ∘ exp(ξ^)) at ξ = 0 with the aff(3) basis (per-point form, see module doc)."""
    X = stats.X
    n = X.shape[0]
    gt = np.eye(4)
    gt[:3, :3], gt[:3, 3] = A, t
    xt = np.concatenate([X, np.ones((n, 1))], axis=1)            # x̃_n
    z = X @ A.T + t
    v = np.einsum("nij,nj->ni", stats.H, z) - stats.g
    E = [basis(k + 1) for k in range(K_AFF)]
    J = np.stack([(xt @ (gt @ Ek).T)[:, :3] for Ek in E], axis=1)  # [n, K, 3]
    grad = np.einsum("ni,nki->k", v, J)
    HJ = np.einsum("nij,nlj->nli", stats.H, J)                    # H_n J_nl
    H = np.einsum("nki,nli->kl", J, HJ)
    for k in range(K_AFF):
        for l in range(K_AFF):
            S = gt @ (0.5 * (E[k] @ E[l] + E[l] @ E[k]))
            H[k, l] += float(np.einsum("ni,ni->", v, (xt @ S.T)[:, :3]))
    return grad, H


def newton(stats, extent: float, newton_max: int = 10):
    """Damped Newton on GA⁺(3) from the E-step transform (the rigid oracle's rules, R11-R13)."""
    A, t = stats.R_E.copy(), stats.t_E.copy()
    q_cur = 0.0
    info = {"newton_iters": 0, "damped": 0, "converged": False}
    for it in range(newton_max):
        grad, H = grad_hess(stats, A, t)
        tr = abs(np.trace(H)) / K_AFF
        mu = 0.0
        accepted = converged = False
        for _ in range(20):
            try:
                L = np.linalg.cholesky(H + mu * np.eye(K_AFF))
            except np.linalg.LinAlgError:
                mu = max(10.0 * mu, 1e-6 * tr)
                continue
            delta = -np.linalg.solve(L.T, np.linalg.solve(L, grad))
            if np.linalg.norm(delta[:9]) < 1e-10 and np.linalg.norm(delta[9:]) < 1e-10 * extent:
                converged = True
                break
            An, tn = compose(A, t, *exp(delta))
            qn = stats.q_rel(An, tn)
            if qn < q_cur:
                A, t, q_cur, accepted = An, tn, qn, True
                break
            mu = max(10.0 * mu, 1e-6 * tr)
        if mu > 0.0:
            info["damped"] += 1
        if converged or not accepted:
            info["converged"] = converged
            break
        info["newton_iters"] = it + 1
    return A, t, q_cur, info


def weighted_affine_lstsq(stats):
    """The unconstrained minimiser of q over all affine maps, by ordinary weighted linear least squares:
    Σ_n (A x_n + t)ᵀ H_n (A x_n + t) - 2 g_nᵀ (A x_n + t) in θ = vec([A | t]) (a textbook pin, reading R24)."""
    X = stats.X
    n = X.shape[0]
    xt = np.concatenate([X, np.ones((n, 1))], axis=1)
    # z_n = Φ_n θ with Φ_n = I_3 ⊗ x̃_nᵀ (row-major θ)
    Phi = np.zeros((n, 3, 12))
    for i in range(3):
        Phi[:, i, 4 * i:4 * i + 4] = xt
    Nm = np.einsum("nai,nab,nbj->ij", Phi, stats.H, Phi)
    rhs = np.einsum("nai,na->i", Phi, stats.g)
    th = np.linalg.solve(Nm, rhs).reshape(3, 4)
    return th[:, :3], th[:, 3]
