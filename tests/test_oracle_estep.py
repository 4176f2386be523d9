"""Pins for the oracle E step (Eq. 1, 2, 5, 9, 10).

Independent references used here:
* brute force of Eq. 5 with an explicit 3×3 Σ_m (numpy inv/det) and Gaussian normaliser (pure loops);
* the paper's matrix form Eq. 9-10 (oracle/matrix_form.py, written separately from the C oracle);
* the isotropic CPD E step (α ≡ 0) written out textbook-style;
* numerical quadrature of the component density (c_m is a normalising constant);
* SPEC worked values for c_m.
"""
import numpy as np
import pytest

import oracle


def _instance(rng, M, N, scale=1.0):
    Y = rng.standard_normal((M, 3)) * scale
    n = rng.standard_normal((M, 3))
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    a = rng.uniform(0, 50, M)
    X = rng.standard_normal((N, 3)) * scale
    R, t = oracle.se3.exp(rng.standard_normal(6) * 0.3)
    return Y, n, a, X, R, t


def _brute_eq5(Y, n, a, X, R, t, s2, w, V, consistent):
    """Eq. 5 per pair with an explicit covariance matrix (pure Python loops)."""
    M, N = Y.shape[0], X.shape[0]
    P = np.zeros((M, N))
    Po = np.zeros(N)
    lnp = np.zeros(N)
    for j in range(N):
        xh = R @ X[j] + t
        dens = np.zeros(M)
        for m in range(M):
            Sinv = (a[m] * np.outer(n[m], n[m]) + np.eye(3)) / s2          # Eq. 2
            Sigma = np.linalg.inv(Sinv)
            if consistent:
                c = 1.0 / ((2 * np.pi) ** 1.5 * np.sqrt(np.linalg.det(Sigma)))
            else:
                c = 1.0 / (2 * np.pi * s2) ** 1.5                          # Eq. 9-10 literal C (no det factor)
            r = xh - Y[m]
            dens[m] = c * np.exp(-0.5 * r @ Sinv @ r)
        mix = (1 - w) / M * dens                                           # (1-w) π(m) p(x|m)
        total = w / V + mix.sum()                                          # Eq. 1 with p_o = 1/V
        P[:, j] = mix / total
        Po[j] = (w / V) / total
        lnp[j] = np.log(total)
    return P, Po, lnp


@pytest.mark.parametrize("w", [0.0, 0.1, 0.7])
@pytest.mark.parametrize("consistent", [True, False])
def test_estep_vs_bruteforce(w, consistent):
    rng = np.random.default_rng(10)
    Y, n, a, X, R, t = _instance(rng, 7, 9)
    s2, V = 0.8, 30.0
    Pb, Pob, lnpb = _brute_eq5(Y, n, a, X, R, t, s2, w, V, consistent)
    P, Po = oracle.posterior(Y, n, a, X, R, t, s2, w, V, consistent)
    np.testing.assert_allclose(P, Pb, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(Po, Pob, rtol=1e-12, atol=1e-15)
    rec = oracle.estep(Y, n, a, X, R, t, s2, w, V, consistent)
    # definitional sums of the pinned P (record layout: include/lsgcpd.h / oracle/lsgcpd_oracle.c)
    d = np.zeros_like(Pb)
    for m in range(7):
        for j in range(9):
            r = R @ X[j] + t - Y[m]
            d[m, j] = (r @ r + a[m] * (n[m] @ r) ** 2) / s2
    np.testing.assert_allclose(rec[:, 0], Pb.sum(0), rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(rec[:, 1:4], Pb.T @ Y, rtol=1e-12, atol=1e-14)
    nn = a[:, None, None] * np.einsum("mi,mj->mij", n, n)
    A = np.einsum("mn,mij->nij", Pb, nn)
    np.testing.assert_allclose(rec[:, 4:10], A[:, [0, 0, 0, 1, 1, 2], [0, 1, 2, 1, 2, 2]], rtol=1e-11, atol=1e-14)
    bvec = (a * np.einsum("mi,mi->m", n, Y))[:, None] * n
    np.testing.assert_allclose(rec[:, 10:13], Pb.T @ bvec, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(rec[:, 13], (Pb * d).sum(0), rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(rec[:, 14], lnpb, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(rec[:, 15], Pob, rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(rec[:, 0] + rec[:, 15], 1.0, rtol=0, atol=1e-14)


@pytest.mark.parametrize("consistent", [True, False])
def test_estep_vs_matrix_form(consistent):
    rng = np.random.default_rng(11)
    Y, n, a, X, R, t = _instance(rng, 40, 50, scale=0.5)
    s2, w, V = 0.3, 0.2, 8.0
    Pm, Pom = oracle.matrix_form.correspondence(Y, n, a, X, R, t, s2, w, V, consistent)
    P, Po = oracle.posterior(Y, n, a, X, R, t, s2, w, V, consistent)
    np.testing.assert_allclose(P, Pm, rtol=1e-11, atol=1e-14)
    np.testing.assert_allclose(Po, Pom, rtol=1e-11, atol=1e-14)


def test_alpha_zero_is_isotropic_cpd():
    # S:316 / SURVEY §8(c).5: α ≡ 0 reduces to the CPD E step with a V-normalised outlier term:
    # P_mn = exp(-||x̂_n - y_m||²/2σ²) / (Σ_k exp(-||x̂_n - y_k||²/2σ²) + (2πσ²)^{3/2} w/(1-w) M/V)
    rng = np.random.default_rng(12)
    Y, n, a, X, R, t = _instance(rng, 30, 25)
    a[:] = 0.0
    s2, w, V = 0.5, 0.3, 20.0
    Xh = X @ R.T + t
    G = np.exp(-((Xh[None, :, :] - Y[:, None, :]) ** 2).sum(-1) / (2 * s2))
    c = (2 * np.pi * s2) ** 1.5 * w / (1 - w) * 30 / V
    Pcpd = G / (G.sum(0, keepdims=True) + c)
    for consistent in (True, False):
        P, _ = oracle.posterior(Y, n, a, X, R, t, s2, w, V, consistent)
        np.testing.assert_allclose(P, Pcpd, rtol=1e-12, atol=1e-15)


def test_normaliser_worked_values():
    # c = (2π)^{-3/2} ≈ 0.063494 at α=0, σ²=1; c = 2(2π)^{-3/2} at α=3.
    # With M = 1, w = 0 and x̂ = y, ln p(x̂) = ln c_m.
    for alpha, c in ((0.0, 0.063494), (3.0, 2 * (2 * np.pi) ** -1.5)):
        rec = oracle.estep(np.zeros((1, 3)), np.array([[0, 0, 1.0]]), np.array([alpha]), np.zeros((1, 3)),
                           np.eye(3), np.zeros(3), 1.0, 0.0, 1.0, True)
        assert np.exp(rec[0, 14]) == pytest.approx(c, rel=1e-5 if alpha == 0 else 1e-14)
        assert rec[0, 0] == 1.0 and rec[0, 15] == 0.0


def test_component_density_integrates_to_one():
    # P:151 "c_m is a normalizing constant": ∫ p(x|m) dx = 1 only with the sqrt(1+α) factor.
    n = np.array([[0.6, 0.0, 0.8]])
    alpha, s2 = 3.0, 0.25
    g = np.linspace(-3.5, 3.5, 141)
    h = g[1] - g[0]
    G = np.stack(np.meshgrid(g, g, g, indexing="ij"), -1).reshape(-1, 3)
    for consistent, expect in ((True, 1.0), (False, 1.0 / np.sqrt(1 + alpha))):
        rec = oracle.estep(np.zeros((1, 3)), n, np.array([alpha]), G, np.eye(3), np.zeros(3), s2, 0.0, 1.0,
                           consistent)
        assert np.exp(rec[:, 14]).sum() * h ** 3 == pytest.approx(expect, rel=1e-6)


def test_sign_and_rigid_invariance():
    rng = np.random.default_rng(13)
    Y, n, a, X, R, t = _instance(rng, 50, 40)
    s2, w, V = 0.4, 0.1, 10.0
    r0 = oracle.estep(Y, n, a, X, R, t, s2, w, V)
    r1 = oracle.estep(Y, -n, a, X, R, t, s2, w, V)                      # S:153 sign of n is irrelevant
    np.testing.assert_allclose(r1, r0, rtol=1e-13, atol=1e-15)
    # rigid conjugation: move the target by T and the pose by T∘g; scalar stats unchanged
    RT, tT = oracle.se3.exp(np.array([0.4, -0.2, 1.0, 2.0, -1.0, 0.5]))
    r2 = oracle.estep(Y @ RT.T + tT, n @ RT.T, a, X, RT @ R, RT @ t + tT, s2, w, V)
    for c in (0, 13, 14, 15):
        np.testing.assert_allclose(r2[:, c], r0[:, c], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(r2[:, 1:4], r0[:, 1:4] @ RT.T + r0[:, :1] * tT, rtol=1e-9, atol=1e-12)


def test_hand_cases():
    # M = N = 1 by hand: P = K/(K+γ)
    y = np.array([[0.1, 0.2, 0.3]])
    x = np.array([[0.3, 0.1, 0.2]])
    n = np.array([[0.0, 0.0, 1.0]])
    alpha, s2, w, V = 2.0, 0.05, 0.25, 3.0
    r = x[0] - y[0]
    d = (r @ r + alpha * r[2] ** 2) / s2
    K = (1 - w) / w * np.sqrt(1 + alpha) * np.exp(-d / 2)
    gamma = (2 * np.pi * s2) ** 1.5 / V
    rec = oracle.estep(y, n, np.array([alpha]), x, np.eye(3), np.zeros(3), s2, w, V)
    assert rec[0, 0] == pytest.approx(K / (K + gamma), rel=1e-14)
    assert rec[0, 13] == pytest.approx(K / (K + gamma) * d, rel=1e-14)
    # near-zero w with a coincident point → P → 1; far point → outlier posterior → 1
    rec = oracle.estep(y, n, np.array([0.0]), y, np.eye(3), np.zeros(3), 1e-2, 1e-9, V)
    assert rec[0, 0] == pytest.approx(1.0, abs=1e-6)
    rec = oracle.estep(y, n, np.array([0.0]), y + 5.0, np.eye(3), np.zeros(3), 1e-2, 0.1, V)
    assert rec[0, 15] == pytest.approx(1.0, abs=1e-12) and rec[0, 0] < 1e-100
    # w = 0 is a pure softmax over components even for far points (no 0/0)
    rec = oracle.estep(np.vstack([y, y + 1]), np.vstack([n, n]), np.zeros(2), y + 1e3, np.eye(3), np.zeros(3),
                       1e-4, 0.0, V)
    assert rec[0, 0] == pytest.approx(1.0, abs=1e-14) and rec[0, 15] == 0.0


def test_uniform_alpha_normaliser_modes_agree_without_outliers():
    # with w = 0 and a common α the sqrt(1+α) factor cancels in Eq. 5
    rng = np.random.default_rng(14)
    Y, n, a, X, R, t = _instance(rng, 20, 15)
    a[:] = 7.0
    r1 = oracle.estep(Y, n, a, X, R, t, 0.3, 0.0, 5.0, True)
    r0 = oracle.estep(Y, n, a, X, R, t, 0.3, 0.0, 5.0, False)
    np.testing.assert_allclose(r1[:, :14], r0[:, :14], rtol=1e-12, atol=1e-15)
    np.testing.assert_allclose(r1[:, 14] - r0[:, 14], 0.5 * np.log(8.0), rtol=1e-12)
