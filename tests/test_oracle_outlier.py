"""Pins for the oracle's outlier-weight estimation (Eq. 7) and confidence filtering
(Eq. 8) — against the paper's defining property, SPEC worked values, special cases that
reduce to the uniform model, and brute force."""
import numpy as np
import pytest

import oracle
from oracle import outlier as ol


def test_wmax_worked_value_and_limits():
    # M=1, π=1, α=0, σ²=1, V=(2π)^{3/2} (so V·c = 1), η = 0.5 → w0 = 0.5
    V = (2.0 * np.pi) ** 1.5
    assert ol.outlier_weight_max(0.5, V, [1.0], [0.0], 1.0) == pytest.approx(0.5, abs=1e-15)
    assert ol.outlier_weight_max(0.0, V, [1.0], [0.0], 1.0) == 0.0
    etas = np.linspace(0, 0.999, 50)
    w = [ol.outlier_weight_max(e, 3.0, [0.3, 0.7], [1.0, 40.0], 0.01) for e in etas]
    assert np.all(np.diff(w) > 0) and w[-1] < 1.0 and ol.outlier_weight_max(1 - 1e-12, 3.0, [1.0], [0.0], 0.01) > 0.99
    Vs = np.linspace(0.1, 10, 20)                                                      # monotone in V
    assert np.all(np.diff([ol.outlier_weight_max(0.2, v, [1.0], [5.0], 0.01) for v in Vs]) > 0)
    with pytest.raises(ValueError):
        ol.outlier_weight_max(1.0, 1.0, [1.0], [0.0], 1.0)


@pytest.mark.parametrize("consistent", [True, False])
def test_eq7_expected_outlier_count_at_the_density_bound(consistent):
    # Eq. 7's defining property: when every p(g*(x_n)|m) equals its bound c_m — every source point at the
    # common centre of all components — w0 = w_max makes Σ_n P(M+1|x_n) = ηN exactly.
    rng = np.random.default_rng(3)
    M, N = 7, 11
    y0 = np.array([0.3, -0.2, 0.5])
    Y = np.tile(y0, (M, 1))
    n = rng.standard_normal((M, 3)); n /= np.linalg.norm(n, axis=1, keepdims=True)
    a = rng.uniform(0, 50, M)
    prior = ol.confidence_prior(rng.uniform(0.1, 1.0, M))
    X = np.tile(y0, (N, 1))
    for eta in (0.05, 0.3, 0.8):
        for s2 in (1e-3, 0.2):
            V = 2.5
            w0 = ol.outlier_weight_max(eta, V, prior, a, s2, consistent)
            rec = oracle.estep_cf(Y, n, a, prior, X, np.full(N, w0), np.eye(3), np.zeros(3), s2, V, consistent)
            assert ol.expected_outliers(rec[:, 15]) == pytest.approx(eta * N, rel=1e-10)


def test_eq8_special_cases():
    # φ ≡ 1 is the uniform model: π = 1/M, w_n = w0, and the E step equals the plain one
    rng = np.random.default_rng(4)
    M, N = 40, 30
    Y = rng.uniform(-1, 1, (M, 3)); X = rng.uniform(-1, 1, (N, 3))
    n = rng.standard_normal((M, 3)); n /= np.linalg.norm(n, axis=1, keepdims=True)
    a = rng.uniform(0, 50, M)
    R, t = oracle.se3.exp(rng.standard_normal(6) * 0.1)
    pi = ol.confidence_prior(np.ones(M))
    wn = ol.point_outlier_weights(0.2, np.ones(N))
    np.testing.assert_allclose(pi, 1.0 / M, rtol=1e-15)
    np.testing.assert_allclose(wn, 0.2, rtol=1e-15)
    a_ = oracle.estep_cf(Y, n, a, pi, X, wn, R, t, 0.05, 6.0)
    b_ = oracle.estep(Y, n, a, X, R, t, 0.05, 0.2, 6.0)
    np.testing.assert_allclose(a_, b_, rtol=1e-12, atol=1e-14)
    # two targets with φ = (1, 0.5) → π = (2/3, 1/3); φ(x_n) = 0 → w_n = 1, all outlier
    np.testing.assert_allclose(ol.confidence_prior([1.0, 0.5]), [2 / 3, 1 / 3], rtol=1e-15)
    assert ol.point_outlier_weights(0.3, [0.0])[0] == 1.0
    wn0 = wn.copy(); wn0[:5] = 1.0
    r = oracle.estep_cf(Y, n, a, pi, X, wn0, R, t, 0.05, 6.0)
    assert np.all(r[:5, 15] == 1.0) and np.all(r[:5, :14] == 0.0)
    np.testing.assert_allclose(r[:5, 14], np.log(1.0 / 6.0), rtol=1e-14)
    np.testing.assert_allclose(r[:, 0] + r[:, 15], 1.0, atol=1e-14)
    with pytest.raises(ValueError):
        ol.confidence_prior(np.zeros(3))


def test_estep_cf_vs_bruteforce():
    # Eq. 1 and Eq. 5 with π(m) and w_n, evaluated with an explicit Σ_m⁻¹, det and Gaussian in pure Python
    rng = np.random.default_rng(5)
    M, N = 6, 5
    Y = rng.uniform(-0.3, 0.3, (M, 3)); X = rng.uniform(-0.3, 0.3, (N, 3))
    n = rng.standard_normal((M, 3)); n /= np.linalg.norm(n, axis=1, keepdims=True)
    a = rng.uniform(0, 30, M)
    pi = ol.confidence_prior(rng.uniform(0.05, 1, M))
    wn = ol.point_outlier_weights(0.1, rng.uniform(0, 1, N))
    R, t = oracle.se3.exp(rng.standard_normal(6) * 0.2)
    s2, V = 0.02, 1.7
    rec = oracle.estep_cf(Y, n, a, pi, X, wn, R, t, s2, V)
    for j in range(N):
        xh = R @ X[j] + t
        dens = []
        for m in range(M):
            Si = (a[m] * np.outer(n[m], n[m]) + np.eye(3)) / s2
            c = np.sqrt(np.linalg.det(Si)) / (2 * np.pi) ** 1.5
            r = xh - Y[m]
            dens.append(c * np.exp(-0.5 * r @ Si @ r))
        dens = np.array(dens)
        px = wn[j] / V + (1 - wn[j]) * np.dot(pi, dens)
        P = (1 - wn[j]) * pi * dens / px
        assert rec[j, 0] == pytest.approx(P.sum(), rel=1e-12)
        np.testing.assert_allclose(rec[j, 1:4], P @ Y, rtol=1e-11, atol=1e-15)
        assert rec[j, 14] == pytest.approx(np.log(px), rel=1e-12)
        assert rec[j, 15] == pytest.approx(wn[j] / V / px, rel=1e-12)


def test_depth_confidence_and_truncation():
    assert ol.depth_confidence(0.4) == pytest.approx(1.0)
    assert ol.depth_confidence(0.8) == pytest.approx(0.25)          # e ∝ z² (c0 = 0)
    z = np.linspace(0.1, 8, 50)
    phi = ol.depth_confidence(z)
    assert np.all(phi <= 1.0) and np.all(np.diff(phi[z >= 0.4]) < 0)
    pts = np.arange(12.0).reshape(4, 3)
    kept, kphi, keep = ol.truncate(pts, [1.0, 0.1, 0.5, 0.05], 0.2)
    assert keep.tolist() == [True, False, True, False] and kept.tolist() == [pts[0].tolist(), pts[2].tolist()]


def test_em_general_model_reduces_to_uniform():
    import synth
    wl = synth.make("tiny")
    tg = oracle.prepare_target(wl.target, wl.knn_k)
    V, ext = oracle.working_volume(wl.target)
    a = oracle.register(tg, wl.source, wl.w, 8, V, ext)
    b = oracle.register(tg, wl.source, wl.w, 8, V, ext, prior=np.full(wl.M, 1.0 / wl.M), phi_x=np.ones(wl.N))
    np.testing.assert_allclose(b["R"], a["R"], atol=1e-10)
    np.testing.assert_allclose(b["sigma2"], a["sigma2"], rtol=1e-8)
    # with η the baseline weight follows σ²_k (c_m ∝ σ^-3): w0_k from the trace matches Eq. 7 at each σ²_k
    c = oracle.register(tg, wl.source, 0.0, 5, V, ext, eta=0.1)
    for s2, w0 in zip(c["trace"]["sigma2"], c["trace"]["w0"]):
        assert w0 == pytest.approx(ol.outlier_weight_max(0.1, V, np.full(wl.M, 1.0 / wl.M), tg["alpha"], s2))
