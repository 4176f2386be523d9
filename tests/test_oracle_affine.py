"""Pins for the oracle M step on the affine group: the matrix exponential
against its power series; ∇/H against central finite differences; the se(3) components of the affine
derivatives against the independently written rigid oracle; the Newton fixed point against ordinary
weighted linear least squares over affine maps; exact recovery of a noiseless affine transform."""
import numpy as np
import pytest

import oracle
from oracle import affine as af, se3


def _stats(rng, M=30, N=40, w=0.1):
    Y = rng.standard_normal((M, 3))
    n = rng.standard_normal((M, 3)); n /= np.linalg.norm(n, axis=1, keepdims=True)
    a = rng.uniform(0, 50, M)
    X = Y[rng.integers(0, M, N)] + 0.2 * rng.standard_normal((N, 3))
    A = np.eye(3) + 0.1 * rng.standard_normal((3, 3))
    t = 0.1 * rng.standard_normal(3)
    s2 = 0.3
    return Y, n, a, X, A, t, s2


def _record(Y, n, a, X, A, t, s2, w=0.1, V=50.0):
    # oracle.estep takes a 3×3 matrix; with a non-orthogonal A it evaluates x̂ = A x + t all the same
    return oracle.estep(Y, n, a, X, A, t, s2, w, V)


def test_affine_exp_and_basis():
    rng = np.random.default_rng(30)
    for _ in range(4):
        xi = 0.5 * rng.standard_normal(12)
        G = af.hat(xi)
        S, term = np.eye(4), np.eye(4)
        for k in range(1, 40):
            term = term @ G / k
            S = S + term
        A, t = af.exp(xi)
        np.testing.assert_allclose(A, S[:3, :3], atol=1e-12)
        np.testing.assert_allclose(t, S[:3, 3], atol=1e-12)
    A, t = af.exp(np.r_[np.zeros(9), 0.3, -0.2, 0.1])
    np.testing.assert_allclose(A, np.eye(3), atol=0)
    np.testing.assert_allclose(t, [0.3, -0.2, 0.1], atol=0)
    # exp of a diagonal generator is a pure scaling e^s
    A, _ = af.exp(np.r_[0.2, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0])
    assert A[0, 0] == pytest.approx(np.exp(0.2), rel=1e-14) and A[1, 1] == 1.0


def test_affine_grad_hess_vs_finite_differences():
    rng = np.random.default_rng(31)
    Y, n, a, X, A, t, s2 = _stats(rng)
    rec = _record(Y, n, a, X, A, t, s2)
    st = oracle.PointStats(X, rec, A, t, s2)
    A1 = A @ (np.eye(3) + 0.05 * rng.standard_normal((3, 3)))
    t1 = t + 0.05 * rng.standard_normal(3)
    g, H = af.grad_hess(st, A1, t1)

    def f(xi):
        return 0.5 * st.q_total(*af.compose(A1, t1, *af.exp(xi)))
    h = 1e-5
    E = np.eye(12)
    gfd = np.array([(f(h * E[k]) - f(-h * E[k])) / (2 * h) for k in range(12)])
    np.testing.assert_allclose(g, gfd, rtol=1e-6, atol=1e-8 * np.abs(gfd).max())
    hh = 1e-4
    Hfd = np.zeros((12, 12))
    for k in range(12):
        gp, _ = af.grad_hess(st, *af.compose(A1, t1, *af.exp(hh * E[k])))
        gm, _ = af.grad_hess(st, *af.compose(A1, t1, *af.exp(-hh * E[k])))
        Hfd[:, k] = (gp - gm) / (2 * hh)
    # the right-derivative Hessian of the group function is the symmetrised Eq. 12 (its FD is not symmetric)
    np.testing.assert_allclose(H, 0.5 * (Hfd + Hfd.T), rtol=1e-5, atol=1e-6 * np.abs(H).max())


def test_affine_derivatives_restricted_to_se3_equal_the_rigid_oracle():
    # the rotation generators of se(3) are skew(e_a) = combinations of the aff(3) generators e_i e_jᵀ; the
    # derivatives are linear (∇) and bilinear (H) in the generator, so L ∇_aff and Lᵀ H_aff L must equal the
    # rigid oracle's ∇ and H, written independently in oracle/mstep.py
    rng = np.random.default_rng(32)
    Y, n, a, X, _, _, s2 = _stats(rng)
    R, t = se3.exp(rng.standard_normal(6) * 0.3)
    rec = _record(Y, n, a, X, R, t, s2)
    st = oracle.PointStats(X, rec, R, t, s2)
    R1, t1 = se3.compose(R, t, *se3.exp(rng.standard_normal(6) * 0.05))
    L = np.zeros((12, 6))
    for k in range(6):
        E = se3.basis(k + 1)
        for m in range(12):
            L[m, k] = np.sum(E * af.basis(m + 1))     # coordinates of E_k in the aff(3) basis
    ga, Ha = af.grad_hess(st, R1, t1)
    gr, Hr = st.grad_hess(R1, t1)
    np.testing.assert_allclose(L.T @ ga, gr, rtol=1e-10, atol=1e-10 * np.abs(gr).max())
    np.testing.assert_allclose(L.T @ Ha @ L, Hr, rtol=1e-10, atol=1e-10 * np.abs(Hr).max())


def test_affine_newton_reaches_the_weighted_least_squares_optimum():
    rng = np.random.default_rng(33)
    Y, n, a, X, A, t, s2 = _stats(rng)
    rec = _record(Y, n, a, X, A, t, s2)
    st = oracle.PointStats(X, rec, A, t, s2)
    A_ls, t_ls = af.weighted_affine_lstsq(st)
    assert np.linalg.det(A_ls) > 0
    A_n, t_n, q, info = af.newton(st, 3.0, newton_max=50)
    np.testing.assert_allclose(A_n, A_ls, atol=1e-8)
    np.testing.assert_allclose(t_n, t_ls, atol=1e-8)
    assert q <= st.q_rel(A_ls, t_ls) + 1e-9 * abs(q)


def test_affine_em_recovers_a_noiseless_affine_transform():
    import synth
    wl = synth.make("tiny_noiseless")
    tg = oracle.prepare_target(wl.target, wl.knn_k)
    V, ext = oracle.working_volume(wl.target)
    A_gt = np.array([[1.08, 0.05, 0.0], [-0.03, 0.95, 0.04], [0.02, 0.0, 1.03]])
    t_gt = np.array([0.02, -0.03, 0.01])
    Xs = ((wl.target.astype(np.float64) - t_gt) @ np.linalg.inv(A_gt).T)   # source = g_gt⁻¹(target)
    out = oracle.register(tg, Xs, 0.1, 80, V, ext, group="affine")
    np.testing.assert_allclose(out["R"], A_gt, atol=1e-6)
    np.testing.assert_allclose(out["t"], t_gt, atol=1e-6 * ext)
