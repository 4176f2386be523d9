"""Pins for the oracle SE(3) M step (§3.5, Eq. 11-13; σ² update P:341).

References: SE(3) textbook identities and power series; central finite differences of the frozen-P
objective; the literal Eq. 11/12 double sums; weighted Procrustes (Kabsch/SVD) for α ≡ 0;
1-D minimisation of Q in σ².
"""
import numpy as np
import pytest

import oracle
from oracle import se3


def test_se3_basics():
    R, v = se3.exp(np.array([0, 0, np.pi / 2, 0, 0, 0]))
    np.testing.assert_allclose(R, [[0, -1, 0], [1, 0, 0], [0, 0, 1]], atol=1e-15)
    R, v = se3.exp(np.array([0, 0, 0, 0.7, 0, 0]))
    np.testing.assert_allclose(R, np.eye(3), atol=0)
    np.testing.assert_allclose(v, [0.7, 0, 0], atol=0)
    E1, E2, E3 = se3.basis(1), se3.basis(2), se3.basis(3)
    np.testing.assert_array_equal(E1 @ E2 - E2 @ E1, E3)
    rng = np.random.default_rng(20)
    for _ in range(5):
        xi = rng.standard_normal(6)
        A = se3.hat(xi)
        S, term = np.eye(4), np.eye(4)
        for k in range(1, 40):
            term = term @ A / k
            S = S + term
        R, t = se3.exp(xi)
        np.testing.assert_allclose(R, S[:3, :3], atol=1e-12)            # S:370 power series
        np.testing.assert_allclose(t, S[:3, 3], atol=1e-12)
        Ri, ti = se3.exp(-xi)
        np.testing.assert_allclose(Ri, R.T, atol=1e-12)
        np.testing.assert_allclose(ti, -R.T @ t, atol=1e-12)
    # branch seam continuity
    d = rng.standard_normal(6)
    d[:3] *= 1e-4 / np.linalg.norm(d[:3])
    Ra, ta = se3.exp(d * (1 - 1e-9))
    Rb, tb = se3.exp(d * (1 + 1e-9))
    np.testing.assert_allclose(Ra, Rb, atol=1e-12)
    np.testing.assert_allclose(ta, tb, atol=1e-12)


def _stats(rng, M=25, N=30, alpha_hi=50.0, w=0.1):
    Y = rng.standard_normal((M, 3))
    n = rng.standard_normal((M, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    a = rng.uniform(0, alpha_hi, M)
    X = Y[rng.integers(0, M, N)] + 0.2 * rng.standard_normal((N, 3))
    R, t = se3.exp(rng.standard_normal(6) * 0.2)
    s2 = 0.3
    rec = oracle.estep(Y, n, a, X, R, t, s2, w, 50.0)
    return Y, n, a, X, R, t, s2, rec


def test_grad_hess_vs_finite_differences():
    rng = np.random.default_rng(21)
    Y, n, a, X, R, t, s2, rec = _stats(rng)
    st = oracle.PointStats(X, rec, R, t, s2)
    Rc, tc = se3.compose(R, t, *se3.exp(rng.standard_normal(6) * 0.05))   # evaluate away from g_E
    grad, H = st.grad_hess(Rc, tc)

    def half_q(xi):
        return 0.5 * st.q_rel(*se3.compose(Rc, tc, *se3.exp(xi)))

    h = 1e-5
    g_fd = np.array([(half_q(h * e) - half_q(-h * e)) / (2 * h) for e in np.eye(6)])
    np.testing.assert_allclose(grad, g_fd, rtol=1e-6, atol=1e-7 * np.abs(grad).max())
    H_fd = np.zeros((6, 6))
    for i in range(6):
        for j in range(6):
            ei, ej = np.eye(6)[i] * 1e-4, np.eye(6)[j] * 1e-4
            H_fd[i, j] = (half_q(ei + ej) - half_q(ei - ej) - half_q(-ei + ej) + half_q(-ei - ej)) / (4e-8)
    np.testing.assert_allclose(H, H_fd, rtol=1e-4, atol=1e-5 * np.abs(H).max())
    np.testing.assert_allclose(H, H.T, atol=1e-12 * np.abs(H).max())


def test_grad_hess_vs_literal_eq11_eq12():
    rng = np.random.default_rng(22)
    Y, n, a, X, R, t, s2, _ = _stats(rng, M=6, N=8)
    Pm, _ = oracle.posterior(Y, n, a, X, R, t, s2, 0.1, 50.0)
    rec = oracle.estep(Y, n, a, X, R, t, s2, 0.1, 50.0)
    st = oracle.PointStats(X, rec, R, t, s2)
    Rc, tc = se3.compose(R, t, *se3.exp(rng.standard_normal(6) * 0.1))
    grad, H = st.grad_hess(Rc, tc)
    g11, H12 = oracle.grad_hess_literal(Pm, Y, n, a, X, Rc, tc, s2)
    # Eq. 11/12 carry a factor 2 and Σ⁻¹ = W/σ² (reading R12): ∇(½q) = σ²/2 ∇_Eq11, H = σ²/2 sym(H_Eq12)
    np.testing.assert_allclose(grad, 0.5 * s2 * g11, rtol=1e-10, atol=1e-13)
    np.testing.assert_allclose(H, 0.5 * s2 * 0.5 * (H12 + H12.T), rtol=1e-10, atol=1e-13)
    assert np.abs(H12 - H12.T).max() > 1e-6                              # Eq. 12 is asymmetric


def _kabsch(X, Ybar, wts):
    mx = (wts[:, None] * X).sum(0) / wts.sum()
    my = (wts[:, None] * Ybar).sum(0) / wts.sum()
    C = ((Ybar - my) * wts[:, None]).T @ (X - mx)
    U, _, Vt = np.linalg.svd(C)
    Dg = np.diag([1, 1, np.sign(np.linalg.det(U @ Vt))])
    R = U @ Dg @ Vt
    return R, my - R @ mx


def test_alpha_zero_mstep_is_weighted_procrustes():
    # with α ≡ 0 the M step has the closed-form CPD/Procrustes solution
    rng = np.random.default_rng(23)
    for trial in range(3):
        Y, n, a, X, R, t, s2, _ = _stats(rng, alpha_hi=0.0)
        rec = oracle.estep(Y, n, np.zeros(len(Y)), X, R, t, s2, 0.1, 50.0)
        Rn, tn, s2n, info = oracle.mstep(X, rec, R, t, s2, extent=5.0, newton_max=50)
        P = rec[:, 0]
        Rk, tk = _kabsch(X, rec[:, 1:4] / P[:, None], P)
        assert se3.rotation_angle(Rn.T @ Rk) < 1e-9
        np.testing.assert_allclose(tn, tk, atol=1e-9)


def test_sigma2_update_is_stationary_point_of_Q():
    rng = np.random.default_rng(24)
    Y, n, a, X, R, t, s2, rec = _stats(rng)
    Rn, tn, s2n, info = oracle.mstep(X, rec, R, t, s2, extent=5.0)
    st = oracle.PointStats(X, rec, R, t, s2)
    q = st.q_total(Rn, tn)
    Pn = rec[:, 0].sum()

    def Q(v):   # σ²-dependent part of Eq. 6 with c_m = sqrt(1+α)/(2πσ²)^{3/2}: Σ P (1.5 ln σ² + τ/(2σ²))
        return Pn * 1.5 * np.log(v) + q / (2 * v)
    lo, hi = 1e-6, 10.0                                                  # golden-section search
    gr = (np.sqrt(5) - 1) / 2
    for _ in range(200):
        c1, c2 = hi - gr * (hi - lo), lo + gr * (hi - lo)
        if Q(c1) < Q(c2):
            hi = c2
        else:
            lo = c1
    assert s2n == pytest.approx(0.5 * (lo + hi), rel=1e-6)   # golden section resolves ~sqrt(eps)
    # single pair, α = 0, ||d||² = 3, P = 1 → σ² = 1
    y = np.zeros((1, 3))
    x = np.array([[1.0, 1.0, 1.0]])
    rec1 = np.zeros((1, 16))
    rec1[0, 0] = 1.0
    rec1[0, 13] = 3.0 / 0.7              # D = ||d||²/σ² at σ² = 0.7
    _, _, s21, _ = oracle.mstep(x, rec1, np.eye(3), np.zeros(3), 0.7, 1.0, newton_max=0)
    assert s21 == pytest.approx(1.0, rel=1e-15)


def test_newton_descends_and_is_stationary_at_optimum():
    rng = np.random.default_rng(25)
    Y, n, a, X, R, t, s2, rec = _stats(rng)
    st = oracle.PointStats(X, rec, R, t, s2)
    Rn, tn, qrel, info = oracle.newton(st, extent=5.0, newton_max=30)
    assert qrel <= 0.0
    g, H = st.grad_hess(Rn, tn)
    assert np.linalg.norm(g) < 1e-8 * max(1.0, np.abs(st.u_E).sum())
    assert np.all(np.linalg.eigvalsh(H) > 0)
