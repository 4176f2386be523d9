"""Oracle M step on SE(3) (§3.5, Eq. 11-13).  TEST INFRASTRUCTURE ONLY.

With P frozen from the E step, the pose part of Q (Eq. 6) is
    Q_pose(g) = q(g) / (2σ²),   q(g) = Σ_n Σ_m P_mn (g(x_n) - y_m)ᵀ W_m (g(x_n) - y_m),   W_m = I + α_m n_m n_mᵀ.
The m-sum is carried by the per-point record: H_n = Σ_m P_mn W_m = P_n I + A_n and
g_n = Σ_m P_mn W_m y_m = Σ_m P_mn y_m + b_n, so (exactly, for z = g(x_n), Δ_n = z - x̂_n):
    Σ_m P_mn (z - y_m)ᵀ W_m (z - y_m) = σ² D_n + 2 Δ_nᵀ u_n + Δ_nᵀ H_n Δ_n,   u_n = H_n x̂_n - g_n.

Gradient and Hessian are right derivatives on the group, g ∘ exp(ξ^) (Eq. 11-12),
of ½q, with J_n = [-[x_n]_× | I] and v_n = Rᵀ(H_n z_n - g_n):
    ∇ = Σ_n [x_n × v_n ; v_n]
    H = Σ_n J_nᵀ (Rᵀ H_n R) J_n + S_n,  S_n = [[½(v xᵀ + x vᵀ) - (v·x) I, -½[v]_×], [½[v]_×, 0]]
S_n is the symmetrised E_iE_j term of Eq. 12; H equals (H_Eq12 + H_Eq12ᵀ)/2 up to the common
factor σ²/2 (tests pin both against the literal Eq. 11/12 double sums and finite differences).

Newton update (Eq. 13), read as δ = -(H + μI)⁻¹∇ with Levenberg damping and a
descent check (readings R11, R13): μ starts at 0; on a failed Cholesky or no decrease of q,
μ ← max(10μ, 1e-6·|tr H|/6); ≤ 20 tries; ≤ newton_max iterations; stop when
||δ_rot|| < 1e-10 and ||δ_trans|| < 1e-10·extent.
σ²: σ²_new = max(floor, q(g_new) / (3 Σ_n P_n)), unchanged when Σ P = 0 (reading R15-R16).
"""
from __future__ import annotations

import numpy as np

from . import se3
from .estep import sym6


class PointStats:
    """Per-point sufficient statistics extracted from an E-step record."""

    def __init__(self, X, rec, R_E, t_E, sigma2):
        self.X = np.ascontiguousarray(X, dtype=np.float64)
        rec = np.asarray(rec, dtype=np.float64)
        self.P = rec[:, 0]
        self.H = self.P[:, None, None] * np.eye(3) + sym6(rec[:, 4:10])
        self.g = rec[:, 1:4] + rec[:, 10:13]
        self.sig2D = sigma2 * rec[:, 13]                 # Σ_m P_mn (x̂-y)ᵀW(x̂-y)
        self.lnp = rec[:, 14]
        self.R_E = np.asarray(R_E, dtype=np.float64)
        self.t_E = np.asarray(t_E, dtype=np.float64)
        self.z_E = self.X @ self.R_E.T + self.t_E
        self.u_E = np.einsum("nij,nj->ni", self.H, self.z_E) - self.g

    def q_rel(self, R, t) -> float:
        """q(g) - q(g_E) = Σ_n 2Δ_nᵀu_n + Δ_nᵀH_nΔ_n."""
        D = self.X @ np.asarray(R).T + np.asarray(t) - self.z_E
        return float((2.0 * (D * self.u_E).sum(axis=1) + np.einsum("ni,nij,nj->n", D, self.H, D)).sum())

    def q_total(self, R, t) -> float:
        return float(self.sig2D.sum()) + self.q_rel(R, t)

    def grad_hess(self, R, t):
        """∇ and H of ½q(g ∘ exp(ξ^)) at ξ = 0 (per-point form)."""
        R = np.asarray(R)
        z = self.X @ R.T + t
        u = np.einsum("nij,nj->ni", self.H, z) - self.g
        v = u @ R                                        # v_n = Rᵀ u_n
        x = self.X
        grad = np.concatenate([np.cross(x, v).sum(axis=0), v.sum(axis=0)])
        K = np.einsum("ai,nab,bj->nij", R, self.H, R)    # Rᵀ H_n R
        n = x.shape[0]
        J = np.zeros((n, 3, 6))
        # -[x]_×
        J[:, 0, 1], J[:, 0, 2] = x[:, 2], -x[:, 1]
        J[:, 1, 0], J[:, 1, 2] = -x[:, 2], x[:, 0]
        J[:, 2, 0], J[:, 2, 1] = x[:, 1], -x[:, 0]
        J[:, :, 3:] = np.eye(3)
        Hs = np.einsum("nai,nab,nbj->ij", J, K, J)
        vx = np.einsum("ni,nj->ij", v, x)
        Hs[:3, :3] += 0.5 * (vx + vx.T) - (v * x).sum() * np.eye(3)
        vs = v.sum(axis=0)
        Hs[:3, 3:] += -0.5 * se3.skew(vs)
        Hs[3:, :3] += 0.5 * se3.skew(vs)
        return grad, Hs


def newton(stats: PointStats, extent: float, newton_max: int = 10):
    """Damped Newton on SE(3) from the E-step pose.  Returns (R, t, q_rel, info)."""
    R, t = stats.R_E.copy(), stats.t_E.copy()
    q_cur = 0.0
    info = {"newton_iters": 0, "damped": 0, "converged": False}
    for it in range(newton_max):
        grad, H = stats.grad_hess(R, t)
        tr = abs(np.trace(H)) / 6.0
        mu = 0.0
        accepted = False
        converged = False
        for _ in range(20):
            A = H + mu * np.eye(6)
            try:
                L = np.linalg.cholesky(A)
            except np.linalg.LinAlgError:
                mu = max(10.0 * mu, 1e-6 * tr)
                continue
            delta = -np.linalg.solve(L.T, np.linalg.solve(L, grad))
            if np.linalg.norm(delta[:3]) < 1e-10 and np.linalg.norm(delta[3:]) < 1e-10 * extent:
                converged = True
                break
            dR, dt = se3.exp(delta)
            Rn, tn = se3.compose(R, t, dR, dt)
            qn = stats.q_rel(Rn, tn)
            if qn < q_cur:
                R, t, q_cur = Rn, tn, qn
                accepted = True
                break
            mu = max(10.0 * mu, 1e-6 * tr)
        if mu > 0.0:
            info["damped"] += 1
        if converged or not accepted:
            info["converged"] = converged
            break
        info["newton_iters"] = it + 1
    return R, t, q_cur, info


def mstep(X, rec, R_E, t_E, sigma2: float, extent: float, newton_max: int = 10, sigma2_floor: float = 0.0,
          group: str = "se3"):
    """One M step: transform by damped Newton on the group (SE(3), or GA⁺(3) for group="affine"),
    then σ² at the new transform."""
    stats = PointStats(X, rec, R_E, t_E, sigma2)
    if group == "affine":
        from .affine import newton as newton_affine
        R, t, q_rel, info = newton_affine(stats, extent, newton_max)
    else:
        R, t, q_rel, info = newton(stats, extent, newton_max)
    sumP = float(stats.P.sum())
    if sumP > 0.0:
        s2 = (float(stats.sig2D.sum()) + q_rel) / (3.0 * sumP)
        s2 = max(sigma2_floor, s2)
    else:
        s2 = sigma2
    info["sumP"] = sumP
    return R, t, s2, info


# ----------------------------------------------------------------------------------------------
# Literal Eq. 11 / Eq. 12 (double sums over m and n with homogeneous forms) — small sizes only.
# ----------------------------------------------------------------------------------------------

def grad_hess_literal(Pmat, Y, normals, alpha, X, R, t, sigma2):
    """∇Q (Eq. 11) and the asymmetric H (Eq. 12) exactly as printed, P:318-332:
        E_i^r Q     = 2 Σ_m Σ_n P_mn (g̃x̃_n - ỹ_m)ᵀ Σ̃_m⁻¹ g̃ E_i x̃_n
        E_i^rE_j^rQ = 2 Σ_m Σ_n P_mn ( x̃_nᵀ E_jᵀ g̃ᵀ Σ̃_m⁻¹ g̃ E_i x̃_n + (g̃x̃_n - ỹ_m)ᵀ Σ̃_m⁻¹ g̃ E_j E_i x̃_n )
    with Σ̃⁻¹ = Σ⁻¹ ⊕ 0."""
    g = se3.homogeneous(R, t)
    E = [se3.basis(i) for i in range(1, 7)]
    M, N = Pmat.shape
    grad = np.zeros(6)
    H = np.zeros((6, 6))
    for m in range(M):
        Si = np.zeros((4, 4))
        Si[:3, :3] = (alpha[m] * np.outer(normals[m], normals[m]) + np.eye(3)) / sigma2
        yt = np.append(Y[m], 1.0)
        for n in range(N):
            p = Pmat[m, n]
            if p == 0.0:
                continue
            xt = np.append(X[n], 1.0)
            r = g @ xt - yt
            gEx = [g @ Ei @ xt for Ei in E]
            for i in range(6):
                grad[i] += 2.0 * p * (r @ Si @ gEx[i])
                for j in range(6):
                    H[i, j] += 2.0 * p * (gEx[j] @ Si @ gEx[i] + r @ Si @ (g @ E[j] @ E[i] @ xt))
    return grad, H
