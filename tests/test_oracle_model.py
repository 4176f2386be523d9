"""Pins for the oracle's target model (§3.1): kNN, κ/normals, α (Eq. 3), V, σ²₀.

Every expected value here comes from the paper's statements, a closed form, brute force or a
geometric special case — never from the oracle itself or from the CUDA path.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_alpha_closed_forms():
    # α → 0 as κ → 1/3, α → α_max as κ → 0; κ=0.1, λ=0.5, α_max=50 → 50·tanh(1.75)
    with open(os.path.join(GOLDEN, "alpha_examples.json")) as f:
        ex = json.load(f)
    for case in ex["cases"]:
        a = oracle.alpha_from_kappa(case["kappa"], case["lambda"], case["alpha_max"])
        assert a == pytest.approx(case["alpha"], abs=case["abs_tol"]), case
    # tanh identity (1-e^{-x})/(1+e^{-x}) = tanh(x/2), x = λ(1/κ - 3)
    k = np.linspace(0.01, 1 / 3, 200)
    np.testing.assert_allclose(oracle.alpha_from_kappa(k, 0.5, 50.0), 50.0 * np.tanh(0.5 * (1 / k - 3) / 2),
                               rtol=1e-13, atol=1e-13)
    assert np.all(np.diff(oracle.alpha_from_kappa(k)) <= 0)     # monotone (saturates at α_max in FP64)
    assert np.all(np.diff(oracle.alpha_from_kappa(k[k > 0.05])) < 0)


def _knn_python(P, k):
    out = []
    for i in range(P.shape[0]):
        d = [(float(((P[j] - P[i]) ** 2).sum()), j) for j in range(P.shape[0])]
        d.sort()
        out.append([j for _, j in d[:k]])
    return np.array(out)


def test_knn_bruteforce_with_ties():
    rng = np.random.default_rng(0)
    P = rng.integers(0, 4, size=(70, 3)).astype(np.float64) * 0.5     # lattice: many exact ties + duplicates
    idx, d2 = oracle.knn(P, 7)
    np.testing.assert_array_equal(idx, _knn_python(P, 7))
    q = np.array([3, 10, 69])
    idx_q, _ = oracle.knn(P, 7, queries=q)
    np.testing.assert_array_equal(idx_q, idx[q])
    assert np.all(np.diff(d2, axis=1) >= 0)


def test_planar_neighbourhood():
    # coplanar points → normal ±z, κ at the clamp floor
    rng = np.random.default_rng(1)
    P = np.column_stack([rng.uniform(-1, 1, (40, 2)), np.zeros(40)])
    idx, _ = oracle.knn(P, 10)
    n, kappa, deg, _ = oracle.local_surface(P, idx)
    assert np.all(np.abs(np.abs(n[:, 2]) - 1.0) < 1e-12)
    assert np.all(kappa == 1e-12)
    assert not deg.any()
    a = oracle.alpha_from_kappa(kappa)
    np.testing.assert_allclose(a, 50.0, rtol=1e-12)               # S:248 flat target → α = α_max


def test_isotropic_and_degenerate_neighbourhoods():
    # equal eigenvalues → κ = 1/3 (octahedron vertices have scatter ∝ I)
    octa = np.array([[1, 0, 0], [-1, 0, 0], [0, 1, 0], [0, -1, 0], [0, 0, 1], [0, 0, -1]], dtype=float)
    idx = np.tile(np.arange(6), (6, 1))
    n, kappa, deg, _ = oracle.local_surface(octa, idx)
    np.testing.assert_allclose(kappa, 1 / 3, rtol=1e-12)
    np.testing.assert_allclose(oracle.alpha_from_kappa(kappa), 0.0, atol=1e-12)
    # all neighbours coincident → degenerate, κ = 1/3, n = (0,0,1)
    P = np.ones((5, 3))
    n, kappa, deg, _ = oracle.local_surface(P, np.tile(np.arange(5), (5, 1)))
    assert deg.all() and np.all(kappa == 1 / 3)
    np.testing.assert_array_equal(n, np.tile([0, 0, 1.0], (5, 1)))


def test_kappa_is_min_rayleigh_quotient():
    # κ = λ_min/trace and n = argmin of the Rayleigh quotient: checked by brute force over directions
    rng = np.random.default_rng(2)
    P = rng.standard_normal((12, 3)) * np.array([1.0, 0.5, 0.1])
    P = P @ oracle.se3.exp(rng.standard_normal(6))[0].T
    idx = np.tile(np.arange(12), (1, 1))
    n, kappa, _, _ = oracle.local_surface(P, idx)
    c = P - P.mean(axis=0)
    C = c.T @ c / 12
    th, ph = np.meshgrid(np.linspace(0, np.pi, 721), np.linspace(0, 2 * np.pi, 1441))
    V = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], -1).reshape(-1, 3)
    rq = np.einsum("vi,ij,vj->v", V, C, V)
    j = np.argmin(rq)
    assert kappa[0] == pytest.approx(rq[j] / np.trace(C), rel=3e-3)   # grid resolution 0.25°
    assert abs(abs(V[j] @ n[0]) - 1.0) < 1e-4 + 1e-5


def test_kappa_rigid_invariance_and_noise_trend():
    rng = np.random.default_rng(3)
    P = np.column_stack([rng.uniform(-1, 1, (300, 2)), 0.02 * rng.standard_normal(300)])
    R, _ = oracle.se3.exp(np.array([0.3, -1.1, 0.7, 0, 0, 0]))
    t1 = oracle.prepare_target(P, 10)
    t2 = oracle.prepare_target(P @ R.T + np.array([5.0, -2.0, 1.0]), 10)
    np.testing.assert_array_equal(t1["knn"], t2["knn"])
    np.testing.assert_allclose(t1["kappa"], t2["kappa"], rtol=1e-7, atol=1e-12)
    # P:402-408 / S:631: mean α decreases as noise grows
    means = []
    for sd in (0.0, 0.01, 0.03, 0.1):
        Q = np.column_stack([rng.uniform(-1, 1, (400, 2)), sd * rng.standard_normal(400)])
        means.append(oracle.prepare_target(Q, 10)["alpha"].mean())
    assert all(a > b for a, b in zip(means, means[1:])), means


def test_working_volume():
    corners = np.array([[x, y, z] for x in (0, 1) for y in (0, 1) for z in (0, 1)], dtype=float)
    V0, ext = oracle.working_volume(corners, margin=0.0)
    assert V0 == pytest.approx(1.0, rel=1e-15) and ext == pytest.approx(np.sqrt(3.0))
    V1, _ = oracle.working_volume(corners, margin=0.1)
    assert V1 == pytest.approx(1.728, rel=1e-14)
    # zero-extent axis floored at the mean nearest-neighbour spacing (grid spacing 0.25)
    g = np.array([[x, y, 0.0] for x in np.arange(5) * 0.25 for y in np.arange(5) * 0.25])
    Vp, _ = oracle.working_volume(g, margin=0.0)
    assert Vp == pytest.approx(1.0 * 1.0 * 0.25, rel=1e-12)


def test_sigma2_init_closed_form_vs_double_sum():
    rng = np.random.default_rng(4)
    X = rng.standard_normal((300, 3)) + 3.0
    Y = rng.standard_normal((250, 3)) * 0.5
    R, t = oracle.se3.exp(rng.standard_normal(6))
    brute = oracle.sum_sq_pairs(X @ R.T + t, Y) / (3 * 300 * 250)
    assert oracle.sigma2_init(X, Y, R, t) == pytest.approx(brute, rel=1e-12)
