"""E-step parity: the sm_100a kernel (through the C ABI) vs the FP64 oracle, element by element.

Inputs: the oracle's prepared target rounded to FP32 (both sides use the same y, n, α), seeded
source clouds, poses {identity, expected} and σ² ∈ {σ²₀, 1e-3, 1e-4, 1e-5}.
Tolerance: 2e-5 of the per-component scale (tests/parity.py), with the local y-scale (x̂, σ²) wherever
the pose is known.  The tensor-core kernel's residual modes are exercised one by one: tile_gate 0 (hi/lo
residual on every tile), the default gate and twice the default gate.
"""
import numpy as np
import pytest

import oracle
from tests.gpu_common import oracle_target32, to_dev, workload
from tests.parity import assert_record_parity, transformed

pytestmark = pytest.mark.gpu

# default: the product's gate; hilo: the hi/lo residual on every tile; wide: twice the default gate (the margin:
# the bar still holds with every tile up to 2× the product's E_tile/σ limit taking the centred residual)
GATES = {"default": None, "hilo": 0.0, "wide": 2 * 24.0}


def _gpu_target(Y, n32, a32):
    import paper_2103_15039_b200 as lsg
    return lsg.pack_target(to_dev(Y), to_dev(n32), to_dev(a32))


def _opts(gate=None, **kw):
    import paper_2103_15039_b200 as lsg
    if gate is not None:
        kw["tile_gate"] = gate
    return lsg.options(**kw)


def _run_pair(Y, n32, a32, X, R, t, s2, w, V, consistent=True, tgt=None):
    import paper_2103_15039_b200 as lsg
    tgt = tgt or _gpu_target(Y, n32, a32)
    rec = lsg.estep(tgt, to_dev(X), R, t, s2, w, V, consistent).cpu().numpy()
    ora = oracle.estep(Y, n32.astype(np.float64), a32.astype(np.float64), X, R, t, s2, w, V, consistent)
    return rec, ora


def _check(rec, ora, Y, a32, X, R, t, s2, what):
    return assert_record_parity(rec, ora, Y, a32, what=what, Xh=transformed(X, R, t), s2=s2)


@pytest.mark.parametrize("name", ["tiny", "object"])
@pytest.mark.parametrize("pose", ["identity", "expected"])
@pytest.mark.parametrize("gate", list(GATES))
def test_estep_parity_sigma_sweep(name, pose, gate):
    wl, n32, a32, V, ext = oracle_target32(name)
    R, t = (np.eye(3), np.zeros(3)) if pose == "identity" else (wl.R_expected, wl.t_expected)
    s2_0 = oracle.sigma2_init(wl.source, wl.target, R, t)
    tgt = _gpu_target(wl.target, n32, a32)
    with _opts(GATES[gate], tc=1):   # the tensor-core kernel at these sizes too
        for s2 in (s2_0, 1e-3, 1e-4, 1e-5):
            rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, s2, wl.w, V, tgt=tgt)
            _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"{name}/{pose}/{gate}/s2={s2:.1e}")
    for s2 in (s2_0, 1e-4):          # and the automatic choice (CUDA cores for tiny)
        rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, s2, wl.w, V, tgt=tgt)
        _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"{name}/{pose}/auto/s2={s2:.1e}")


@pytest.mark.parametrize("w", [0.0, 1e-6, 0.5, 0.9])
@pytest.mark.parametrize("consistent", [True, False])
def test_estep_parity_outlier_weight_and_normaliser(w, consistent):
    # w = 0 (pure softmax, running-max path) and tiny w (running max below the fixed-path threshold)
    wl, n32, a32, V, ext = oracle_target32("tiny")
    R, t = wl.R_expected, wl.t_expected
    for s2 in (1e-2, 1e-4):
        rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, s2, w, V, consistent)
        _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"w={w} consistent={consistent} s2={s2}")
        np.testing.assert_allclose(rec[:, 0] + rec[:, 15], 1.0, atol=2e-6)


@pytest.mark.parametrize("tc", ["auto", "1"])
@pytest.mark.parametrize("M,N", [(1, 1), (3, 7), (63, 65), (64, 512), (257, 513), (1000, 1), (2, 5000),
                                 (130, 769)])
def test_estep_ragged_and_tiny_sizes(M, N, tc):
    # also with the tensor-core kernel forced (tc=1) on sizes below its automatic threshold: a single partial
    # tile, a single partial 768-point block, more CTAs than units
    rng = np.random.default_rng(M * 7919 + N)
    Y = rng.uniform(-1, 1, (M, 3)).astype(np.float32)
    n = rng.standard_normal((M, 3))
    n32 = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    a32 = rng.uniform(0, 50, M).astype(np.float32)
    X = rng.uniform(-1, 1, (N, 3)).astype(np.float32)
    R, t = oracle.se3.exp(rng.standard_normal(6) * 0.1)
    for gate in (("default", "hilo", "wide") if tc == "1" else ("default",)):
        with _opts(GATES[gate], **({"tc": 1} if tc == "1" else {})):
            for w in (0.0, 0.2):
                rec, ora = _run_pair(Y, n32, a32, X, R, t, 0.05, w, 8.0)
                _check(rec, ora, Y, a32, X, R, t, 0.05, f"M={M} N={N} w={w} {gate}")


@pytest.mark.parametrize("tc", ["auto", "1"])
def test_estep_far_points_and_large_coordinates(tc):
    # LiDAR-like magnitudes (|x| ~ 100 m) at small σ²: the hi/lo split and the tile centres keep r accurate
    rng = np.random.default_rng(5)
    M, N = 700, 900
    Y = (rng.uniform(-1, 1, (M, 3)) * np.array([100.0, 100.0, 5.0]) + 50.0).astype(np.float32)
    n32 = np.tile(np.array([[0, 0, 1.0]], np.float32), (M, 1))
    a32 = np.full(M, 40.0, np.float32)
    X = (Y[rng.integers(0, M, N)] + 0.01 * rng.standard_normal((N, 3))).astype(np.float32)
    X[:50] += 1000.0                                             # outliers far from everything
    with _opts(None, **({"tc": 1} if tc == "1" else {})):
        for w in (0.0, 0.1):
            rec, ora = _run_pair(Y, n32, a32, X, np.eye(3), np.zeros(3), 1e-4, w, 2e5)
            _check(rec, ora, Y, a32, X, np.eye(3), np.zeros(3), 1e-4, f"far/large w={w} tc={tc}")


@pytest.mark.parametrize("halves", ["auto", "1"])
@pytest.mark.parametrize("gate", list(GATES))
def test_estep_sampled_parity_at_full_scale(halves, gate):
    # the scale config at full size (M = N = 524,288, the bench's launch configuration): oracle on a sample of
    # source points against every target.  The 84 MB tensor-core section is swept in two halves by default;
    # halves=1 keeps one sweep
    import paper_2103_15039_b200 as lsg
    wl = workload("scale")
    rng = np.random.default_rng(11)
    Y = wl.target
    # seeded annotation: random unit n and α on both sides (the oracle's prepare on 524k targets is slow)
    n = rng.standard_normal(Y.shape)
    n32 = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    a32 = rng.uniform(0, 50, Y.shape[0]).astype(np.float32)
    V, _ = oracle.working_volume(Y)
    tgt = _gpu_target(Y, n32, a32)
    Xd = to_dev(wl.source)
    # 8,192 sampled source points (about 1.6 % of the source, all 8,192 tiles against each) for the
    # product configuration (default gate, two halves); 192 for the other residual modes and the one-sweep form
    nsamp = 8192 if (gate == "default" and halves == "auto") else 192
    idx = np.sort(rng.choice(wl.N, nsamp, replace=False))
    R, t = wl.R_expected, wl.t_expected
    s2_0 = oracle.sigma2_init(wl.source, Y, R, t)
    kw = {} if halves == "auto" else {"halves": 1}
    with _opts(GATES[gate], **kw):
        for s2 in (s2_0, 1e-3, 1e-5):     # σ²₀: every target contributes (longest FP32 sums)
            rec = lsg.estep(tgt, Xd, R, t, s2, wl.w, V).cpu().numpy()[idx]
            ora = oracle.estep(Y, n32.astype(np.float64), a32.astype(np.float64), wl.source[idx], R, t, s2, wl.w, V)
            _check(rec, ora, Y, a32, wl.source[idx], R, t, s2, f"scale sampled {gate} halves={halves} s2={s2}")


@pytest.mark.parametrize("name,gate", [("rgbd", "default"), ("rgbd", "wide"), ("lidar", "default")])
def test_estep_full_record_parity(name, gate):
    # the rgbd (~75k × 77k, 10 % outliers) and lidar (126k × 126k, 100 m outlier box) configs at full size,
    # EVERY source point's record against the oracle, with the oracle's own prepared target (its normals and
    # α), at σ²₀, 1e-3 and the converged σ² of the golden trajectory (tests/golden/<name>_oracle.json)
    import json
    import os
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32(name)
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", f"{name}_oracle.json")))
    tgt = _gpu_target(wl.target, n32, a32)
    Xd = to_dev(wl.source)
    R, t = wl.R_expected, wl.t_expected
    s2_0 = oracle.sigma2_init(wl.source, wl.target, R, t)
    with _opts(GATES[gate]):
        for s2 in (s2_0, 1e-3, float(g["sigma2"])):
            rec = lsg.estep(tgt, Xd, R, t, s2, wl.w, V).cpu().numpy()
            ora = oracle.estep(wl.target, n32.astype(np.float64), a32.astype(np.float64), wl.source, R, t, s2, wl.w, V)
            _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"{name} full record {gate} s2={s2:.3e}")


def test_estep_invalid_arguments_raise():
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    tgt = _gpu_target(wl.target, n32, a32)
    X = to_dev(wl.source)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.estep(tgt, X, np.eye(3), np.zeros(3), -1.0, 0.1, V)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.estep(tgt, X, np.eye(3), np.zeros(3), 1e-3, 1.0, V)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.estep(tgt, X, 2 * np.eye(3), np.zeros(3), 1e-3, 0.1, V)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.estep(tgt, X, np.eye(3), np.array([np.nan, 0, 0]), 1e-3, 0.1, V)


def test_estep_target_mismatch_gives_nan_record():
    # the header check runs on the device (no host sync): a wrong M, or a buffer that is not a prepared
    # target, leaves the record all NaN instead of reading past the target
    import ctypes
    import torch
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    tgt = _gpu_target(wl.target, n32, a32)
    X = to_dev(wl.source)
    L = lsg.lib()
    dp = ctypes.POINTER(ctypes.c_double)
    R = np.eye(3).ravel().copy()
    t = np.zeros(3)
    for M, buf in ((wl.M + 1, tgt.buf), (wl.M - 1, tgt.buf), (wl.M, torch.zeros_like(tgt.buf))):
        ws = torch.empty(L.lsgcpd_estep_workspace_bytes(M, wl.N), dtype=torch.uint8, device="cuda")
        rec = torch.zeros((wl.N, 16), dtype=torch.float32, device="cuda")
        rc = L.lsgcpd_estep(buf.data_ptr(), M, X.data_ptr(), wl.N, R.ctypes.data_as(dp), t.ctypes.data_as(dp),
                            1e-3, 0.1, V, 1, rec.data_ptr(), ws.data_ptr(), ws.numel(),
                            ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        assert rc == 0
        assert torch.isnan(rec).all().item(), f"M={M}"


def test_pack_normalises_normals_and_isotropic_zero_normals():
    # non-unit normals are normalised by the pack (same record as unit normals); a zero normal makes the
    # component isotropic (α := 0), so the record equals the oracle's with α_m = 0 there
    wl, n32, a32, V, ext = oracle_target32("tiny")
    R, t = wl.R_expected, wl.t_expected
    scaled = (n32 * np.linspace(0.3, 3.0, wl.M, dtype=np.float32)[:, None]).astype(np.float32)
    rec_u, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, 1e-3, wl.w, V)
    rec_s, _ = _run_pair(wl.target, scaled, a32, wl.source, R, t, 1e-3, wl.w, V)
    _check(rec_s, ora, wl.target, a32, wl.source, R, t, 1e-3, "scaled normals")
    np.testing.assert_allclose(rec_s, rec_u, rtol=2e-5, atol=1e-6)
    nz = n32.copy()
    nz[::7] = 0.0
    a_eff = a32.copy()
    a_eff[::7] = 0.0
    import paper_2103_15039_b200 as lsg
    rec = lsg.estep(_gpu_target(wl.target, nz, a32), to_dev(wl.source), R, t, 1e-3, wl.w, V).cpu().numpy()
    ora0 = oracle.estep(wl.target, n32.astype(np.float64), a_eff.astype(np.float64), wl.source, R, t, 1e-3, wl.w, V)
    _check(rec, ora0, wl.target, a_eff, wl.source, R, t, 1e-3, "zero normals -> isotropic")


@pytest.mark.parametrize("variant", range(3))
def test_estep_every_cuda_core_configuration(variant):
    # every compiled CUDA-core configuration (768 / 512 / 64-point blocks), tensor cores disabled
    wl, n32, a32, V, ext = oracle_target32("tiny")
    R, t = wl.R_expected, wl.t_expected
    with _opts(None, tc=0, estep_variant=variant):
        for w in (0.0, 0.1):
            rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, 1e-4, w, V)
            _check(rec, ora, wl.target, a32, wl.source, R, t, 1e-4, f"variant {variant} w={w}")


@pytest.mark.parametrize("tc", ["1", "0"])
@pytest.mark.parametrize("gate", list(GATES))
def test_estep_tensor_core_and_cuda_core_paths(tc, gate):
    # default path = tcgen05 kernel (fixed max) + CUDA-core kernel (running max), each residual mode; tc=0
    # (CUDA cores only)
    if tc == "0" and gate != "default":
        pytest.skip("the gate applies to the tensor-core kernel only")
    with _opts(GATES[gate], tc=int(tc)):
        for name in ("tiny", "object"):
            wl, n32, a32, V, ext = oracle_target32(name)
            R, t = wl.R_expected, wl.t_expected
            for w, s2 in ((wl.w, 1e-3), (wl.w, 1e-5), (0.0, 1e-4)):
                rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, s2, w, V)
                _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"tc={tc} {gate} {name} w={w} s2={s2}")


@pytest.mark.parametrize("tc", ["1", "0"])
def test_estep_literal_normaliser_on_both_paths(tc):
    # Eq. 9-10 literal normaliser (reading R1, consistent = 0) through the tensor-core kernel's kLiteral
    # instantiation (forced) and the CUDA-core one, at a size with many tiles and a ragged tail
    wl, n32, a32, V, ext = oracle_target32("object")
    R, t = wl.R_expected, wl.t_expected
    with _opts(None, tc=int(tc)):
        for s2 in (1e-3, 1e-5):
            rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, s2, wl.w, V, False)
            _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"literal tc={tc} s2={s2}")


def test_estep_running_max_path_sampled_at_full_size():
    # w = 0 (pure softmax: the per-point running-max CUDA-core kernel) at the rgbd config's full size
    import paper_2103_15039_b200 as lsg
    wl = workload("rgbd")
    rng = np.random.default_rng(12)
    Y = wl.target
    n = rng.standard_normal(Y.shape)
    n32 = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    a32 = rng.uniform(0, 50, Y.shape[0]).astype(np.float32)
    V, _ = oracle.working_volume(Y)
    tgt = _gpu_target(Y, n32, a32)
    idx = np.sort(rng.choice(wl.N, 128, replace=False))
    R, t = wl.R_expected, wl.t_expected
    for s2 in (1e-2, 1e-4):
        rec = lsg.estep(tgt, to_dev(wl.source), R, t, s2, 0.0, V).cpu().numpy()[idx]
        ora = oracle.estep(Y, n32.astype(np.float64), a32.astype(np.float64), wl.source[idx], R, t, s2, 0.0, V)
        _check(rec, ora, Y, a32, wl.source[idx], R, t, s2, f"rgbd w=0 s2={s2}")
        np.testing.assert_allclose(rec[:, 0], 1.0, atol=2e-6)


def test_tile_centres_exact_on_zero_crossing_and_offset_axes():
    # the pack keeps a tile centre c_a only if every y_a - c_a of the tile is exact in FP32 (else c_a = 0): an axis
    # whose values cross zero with tiny magnitudes must fall back to c_a = 0, an axis far from zero keeps its
    # centre; the E step stays within the bar with every tile centred (gate 2 × default) and with the hi/lo path
    import torch
    rng = np.random.default_rng(17)
    M, N = 2048, 1500
    Y = np.stack([rng.uniform(-1e-3, 1e-3, M), 1e4 + rng.uniform(0.0, 1.0, M), rng.uniform(-5.0, 5.0, M)], 1)
    Y = Y.astype(np.float32)
    n = rng.standard_normal((M, 3))
    n32 = (n / np.linalg.norm(n, axis=1, keepdims=True)).astype(np.float32)
    a32 = rng.uniform(0, 50, M).astype(np.float32)
    X = (Y[rng.integers(0, M, N)] + 0.01 * rng.standard_normal((N, 3))).astype(np.float32)
    tgt = _gpu_target(Y, n32, a32)
    M_pad = (M + 255) // 256 * 256
    off = 256 + M_pad * 16 * 4
    raw = tgt.buf[off: off + (M_pad // 64) * 10240].view(torch.float32).reshape(M_pad // 64, 2560).cpu().numpy()
    c = np.stack([raw[:, 14], raw[:, 15], raw[:, 30]], 1)
    assert np.any(c[:, 0] == 0.0), "no zero-crossing tile fell back to c_x = 0"
    assert np.all(c[:, 1] > 9999.0), "the offset axis lost its centre"
    R, t = np.eye(3), np.zeros(3)
    for gate in ("wide", "hilo"):
        with _opts(GATES[gate], tc=1):
            for s2 in (1e-2, 1e-4):
                rec, ora = _run_pair(Y, n32, a32, X, R, t, s2, 0.1, 1e3, tgt=tgt)
                _check(rec, ora, Y, a32, X, R, t, s2, f"zero-crossing/offset {gate} s2={s2}")


def _morton_order(X):
    # a plain Z-order of the points (test-side, independent of the library's own source ordering)
    lo, hi = X.min(0), X.max(0)
    q = np.floor((X - lo) / max(float((hi - lo).max()), 1e-30) * 1023.0).astype(np.uint64)
    key = np.zeros(len(X), np.uint64)
    for b in range(10):
        for a in range(3):
            key |= ((q[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + a)
    return np.argsort(key, kind="stable")


@pytest.mark.parametrize("name", ["object", "lidar"])
def test_estep_far_rule_on_spatially_ordered_sources(name):
    # the far-point rule (a warp whose points are all >= 2 R_tile from a tile's centre takes the centred residual)
    # only fires when a warp's points are close together: Z-ordered sources.  Checked with the tile gate off, so
    # that every centred tile comes from the rule, and with the product gates; object full records, lidar
    # sampled, at the initial, intermediate and converged σ²
    wl, n32, a32, V, ext = oracle_target32(name)
    X = wl.source[_morton_order(wl.source)]
    R, t = wl.R_expected, wl.t_expected
    tgt = _gpu_target(wl.target, n32, a32)
    idx = np.arange(len(X)) if name == "object" else np.sort(np.random.default_rng(8).choice(len(X), 3000, replace=False))
    import paper_2103_15039_b200 as lsg
    Xd = to_dev(X)
    for s2 in (oracle.sigma2_init(X, wl.target, R, t), 1e-3, 1e-4):
        ora = oracle.estep(wl.target, n32.astype(np.float64), a32.astype(np.float64), X[idx], R, t, s2, wl.w, V)
        for opts in ({"tile_gate": 0.0, "far_rule": 1}, {"far_rule": 1}):
            with lsg.options(tc=1, **opts):
                rec = lsg.estep(tgt, Xd, R, t, s2, wl.w, V).cpu().numpy()[idx]
            assert_record_parity(rec, ora, wl.target, a32, what=f"{name} far rule {opts} s2={s2:.1e}",
                                 Xh=transformed(X[idx], R, t), s2=s2)
        if s2 == 1e-3 and name == "lidar":   # the rule fires: with the gate off it changes some records' rounding
            # (object's tiles around the origin often keep c_a = 0 on an axis — y - c would not be exact — so
            # their R_tile is large and the rule rarely holds there)
            with lsg.options(tc=1, tile_gate=0.0, far_rule=0):
                hilo = lsg.estep(tgt, Xd, R, t, s2, wl.w, V).cpu().numpy()
            with lsg.options(tc=1, tile_gate=0.0, far_rule=1):
                far = lsg.estep(tgt, Xd, R, t, s2, wl.w, V).cpu().numpy()
            assert not np.array_equal(hilo, far), "the far-point rule never fired"



def test_estep_literal_normaliser_with_the_centred_residual():
    # the Eq. 9-10 literal normaliser (kLiteral instantiation) on tiles that take the tile-centred residual:
    # object at σ²₀ and σ² = 0.05, where E_tile / σ is under the default gate
    wl, n32, a32, V, ext = oracle_target32("object")
    R, t = wl.R_expected, wl.t_expected
    s2_0 = oracle.sigma2_init(wl.source, wl.target, R, t)
    tgt = _gpu_target(wl.target, n32, a32)
    with _opts(None, tc=1):
        for s2 in (s2_0, 0.05):
            rec, ora = _run_pair(wl.target, n32, a32, wl.source, R, t, s2, wl.w, V, False, tgt=tgt)
            _check(rec, ora, wl.target, a32, wl.source, R, t, s2, f"literal centred s2={s2:.3g}")
