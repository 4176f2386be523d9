"""Registration parity (the north-star bar): final R within 1e-4 rad and t within 1e-4·extent of the
FP64 oracle on the same seeded inputs, plus EM invariants on the GPU path."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import se3
from tests.gpu_common import oracle_target32, to_dev, workload

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _pack(wl, n32, a32):
    import paper_2103_15039_b200 as lsg
    return lsg.pack_target(to_dev(wl.target), to_dev(n32), to_dev(a32))


def _close(R, t, R_ref, t_ref, extent, tol=1e-4):
    ang = se3.rotation_angle(np.asarray(R).T @ np.asarray(R_ref))
    dt = np.linalg.norm(np.asarray(t) - np.asarray(t_ref))
    assert ang <= tol, f"rotation differs by {ang:.3e} rad"
    assert dt <= tol * extent, f"translation differs by {dt:.3e} (extent {extent:.3f})"
    return ang, dt


def test_register_tiny_vs_oracle_same_target():
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    tgt = _pack(wl, n32, a32)
    gpu = lsg.register(tgt, to_dev(wl.source), wl.iters, w=wl.w, volume=V, traces=True)
    ora = oracle.register({"Y": wl.target.astype(np.float64), "normals": n32.astype(np.float64),
                           "alpha": a32.astype(np.float64)}, wl.source, wl.w, wl.iters, V, ext)
    assert gpu["iters"] == wl.iters and gpu["status"] == 0
    _close(gpu["R"], gpu["t"], ora["R"], ora["t"], ext)
    np.testing.assert_allclose(gpu["sigma2_trace"], ora["trace"]["sigma2"], rtol=1e-3)
    np.testing.assert_allclose(gpu["nll"], ora["trace"]["nll"], rtol=1e-5, atol=1e-3)


def test_register_tiny_end_to_end_gpu_prepared():
    import paper_2103_15039_b200 as lsg
    wl = workload("tiny")
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    gpu = lsg.register(tgt, to_dev(wl.source), wl.iters, w=wl.w)
    ora = oracle.register_workload(wl)
    _close(gpu["R"], gpu["t"], ora["R"], ora["t"], ora["extent"])


def test_register_noiseless_exact_recovery():
    # BJ north star: source = g_gt(target points), no noise → the registration returns g_gt⁻¹.
    # tiny from identity (30°); object from a start 10° off the answer about x (its torus/plane scene is
    # nearly symmetric about z: from identity, or from 10° about z, EM — oracle included — stalls in z).
    import paper_2103_15039_b200 as lsg
    for name, R0, t0 in (("tiny_noiseless", None, None), ("object_noiseless", "near", "near")):
        wl = workload(name)
        if R0 == "near":
            dR, dt = se3.exp(np.array([np.deg2rad(10.0), 0.0, 0.0, 0.02, -0.01, 0.0]))
            R0, t0 = se3.compose(wl.R_expected, wl.t_expected, dR, dt)
        tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
        gpu = lsg.register(tgt, to_dev(wl.source), 60, w=wl.w, R0=R0, t0=t0)
        _close(gpu["R"], gpu["t"], wl.R_expected, wl.t_expected, tgt.extent, tol=1e-5)


@pytest.mark.parametrize("name", ["object", "rgbd", "lidar"])
def test_register_full_size_vs_golden(name):
    # whole registrations at BASELINE.json's full sizes, GPU-prepared target, against the FP64 oracle's own
    # full pipeline (prepare → V → σ²₀ → EM), run offline by oracle/make_golden.py (oracle only)
    import paper_2103_15039_b200 as lsg
    from oracle.make_golden import digest
    path = os.path.join(GOLDEN, f"{name}_oracle.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    g = json.load(open(path))
    wl = workload(name)
    assert (digest(wl.target), digest(wl.source)) == (g["target_sha"], g["source_sha"]), "inputs changed"
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    assert tgt.volume == pytest.approx(g["V"], rel=1e-6)
    gpu = lsg.register(tgt, to_dev(wl.source), g["iters"], w=wl.w, traces=True)
    assert gpu["status"] == 0 and gpu["iters"] == g["iters"]
    _close(gpu["R"], gpu["t"], np.array(g["R"]), np.array(g["t"]), g["extent"])
    # final σ² to 2e-5 relative (achieved in round 1: 5e-8 / 5e-6 / 9e-7, profiles/r01k_golden_errors.txt) and
    # the whole σ² trace to 2e-4 (lidar: 9e-5, r02i)
    assert gpu["sigma2"] == pytest.approx(g["sigma2"], rel=2e-5)
    np.testing.assert_allclose(gpu["sigma2_trace"], np.array(g["sigma2_trace"])[: len(gpu["sigma2_trace"])], rtol=2e-4)


def test_register_nll_monotone_and_deterministic():
    import paper_2103_15039_b200 as lsg
    wl = workload("object")
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    reg = lsg.Registrar(tgt, to_dev(wl.source), 40)
    a = reg(w=wl.w, traces=True)
    b = reg(w=wl.w, traces=True)
    nll = a["nll"]
    assert np.all(np.diff(nll) <= 1e-5 * np.abs(nll).max()), np.diff(nll).max()
    assert np.array_equal(a["R"], b["R"]) and np.array_equal(a["t"], b["t"]) and a["sigma2"] == b["sigma2"]


def test_register_no_mass_and_invalid():
    import paper_2103_15039_b200 as lsg
    wl = workload("tiny")
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    far = to_dev((wl.source + 1e4).astype(np.float32))
    out = lsg.register(tgt, far, 10, w=0.5, sigma2_init=1e-6, check=False)
    assert out["status"] == -5 and out["iters"] == 3
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.register(tgt, to_dev(wl.source), 5, w=1.0)


def test_register_degenerate_and_minimal_inputs():
    # SURVEY §4 fault injection: non-finite coordinates → EINVAL; collinear target (two zero-extent axes)
    # prepares with the floored volume; the minimal problem (M = 3 with k = 3, N = 1) runs
    import paper_2103_15039_b200 as lsg
    wl = workload("tiny")
    bad = wl.target.copy()
    bad[5, 1] = np.nan
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.prepare_target(to_dev(bad), wl.knn_k)
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    src = wl.source.copy()
    src[7, 2] = np.inf
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.register(tgt, to_dev(src), 5, w=wl.w)
    line = np.stack([np.linspace(0, 1, 40), np.zeros(40), np.zeros(40)], axis=1).astype(np.float32)
    lt = lsg.prepare_target(to_dev(line), 10)
    V, _ = oracle.working_volume(line)
    assert lt.volume == pytest.approx(V, rel=1e-6)
    out = lsg.register(lt, to_dev(line[:20] + np.float32(0.01)), 10, w=0.1)
    assert out["status"] == 0 and np.all(np.isfinite(out["R"]))
    tri = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    t3 = lsg.prepare_target(to_dev(tri), 3)
    one = lsg.register(t3, to_dev(np.array([[0.3, 0.3, 0.05]], np.float32)), 5, w=0.1)
    assert one["iters"] == 5 and np.all(np.isfinite(one["t"]))


def test_register_tolerance_stops_early_and_matches_a_fixed_count():
    # tol > 0 (lsgcpd_em_params.tol): stop once |Δσ²|/σ² and the pose step fall below tol; the result is
    # exactly the fixed-count registration with that many iterations (the stop only deactivates the loop)
    import paper_2103_15039_b200 as lsg
    wl = workload("tiny")
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    X = to_dev(wl.source)
    early = lsg.register(tgt, X, 200, w=wl.w, tol=1e-3)
    assert 1 < early["iters"] < 200 and early["status"] == 0
    fixed = lsg.register(tgt, X, early["iters"], w=wl.w)
    np.testing.assert_array_equal(early["R"], fixed["R"])
    np.testing.assert_array_equal(early["t"], fixed["t"])
    assert early["sigma2"] == fixed["sigma2"]


@pytest.mark.parametrize("name,conf", [("tiny", False), ("object", True)])
def test_fused_em_tail_equals_separate_kernels(name, conf):
    # N ≤ 2^17: merge + moments + Newton run as one kernel (em_tail_kernel); LSGCPD_NO_FUSE=1 selects the
    # separate merge / moments / Newton kernels.  Same records, different FP64 summation order of the moments:
    # the registrations agree to FP64 rounding, with and without per-point confidence weights.
    import paper_2103_15039_b200 as lsg
    wl = workload(name)
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    phi = to_dev(np.random.default_rng(2).uniform(0.3, 1.0, wl.N).astype(np.float32)) if conf else None
    kw = dict(w=wl.w, traces=True, src_conf=phi) if conf else dict(w=wl.w, traces=True)
    fused = lsg.register(tgt, to_dev(wl.source), 30, **kw)
    with lsg.options(no_fuse=1):
        sep = lsg.register(tgt, to_dev(wl.source), 30, **kw)
    assert fused["iters"] == sep["iters"] == 30
    _close(fused["R"], fused["t"], sep["R"], sep["t"], tgt.extent, tol=1e-9)
    np.testing.assert_allclose(fused["sigma2_trace"], sep["sigma2_trace"], rtol=1e-9)
    np.testing.assert_allclose(fused["nll"], sep["nll"], rtol=1e-10)


def test_graph_cache_replay_and_update_match_fresh_graphs():
    # lsgcpd_register keeps the instantiated EM-iteration graph of recent calls: a repeated call replays it, a
    # call with other buffers of the same sizes updates it in place (cudaGraphExecUpdate).  Both must give
    # exactly what a freshly captured graph gives (LSGCPD_GRAPH_CACHE=0).
    import paper_2103_15039_b200 as lsg
    import synth
    wls = synth.make_batch(3, 800, seed=21)
    probs = []
    for w in wls:
        tgt = lsg.prepare_target(to_dev(w.target), w.knn_k)
        probs.append(lsg.Registrar(tgt, to_dev(w.source), 25))
    cached = [p(w=0.1) for p in probs] + [probs[0](w=0.1), probs[1](w=0.2)]
    with lsg.options(graph_cache=0):
        fresh = [p(w=0.1) for p in probs] + [probs[0](w=0.1), probs[1](w=0.2)]
    for a, b in zip(cached, fresh):
        assert a["iters"] == b["iters"] == 25
        np.testing.assert_array_equal(a["R"], b["R"])
        np.testing.assert_array_equal(a["t"], b["t"])
        assert a["sigma2"] == b["sigma2"]


@pytest.mark.parametrize("name", ["object_eta", "object_affine"])
def test_register_object_extensions_vs_golden(name):
    # whole object registrations with one model extension — w from the outlier ratio η = 0.1 (Eq. 7,
    # NEXT-1) or the affine group (NEXT-4) — against the oracle's full pipeline
    # (oracle/make_golden.py); for the affine group "R" is the linear part A, compared by ‖A - A_ref‖
    import paper_2103_15039_b200 as lsg
    from oracle.make_golden import digest
    g = json.load(open(os.path.join(GOLDEN, f"{name}_oracle.json")))
    wl = workload("object")
    assert (digest(wl.target), digest(wl.source)) == (g["target_sha"], g["source_sha"]), "inputs changed"
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    kw = {"eta": g["extension"]["eta"]} if "eta" in g["extension"] else {"w": wl.w, "group": "affine"}
    gpu = lsg.register(tgt, to_dev(wl.source), g["iters"], **kw)
    assert gpu["status"] == 0 and gpu["iters"] == g["iters"]
    if name == "object_affine":
        assert np.abs(np.asarray(gpu["R"]) - np.array(g["R"])).max() <= 1e-4
        assert np.linalg.norm(np.asarray(gpu["t"]) - np.array(g["t"])) <= 1e-4 * g["extent"]
    else:
        _close(gpu["R"], gpu["t"], np.array(g["R"]), np.array(g["t"]), g["extent"])
    # σ² to 2e-4 relative: with η the converged σ² is 1e-5 (σ ≈ 3e-3, the E-step weights at their most peaked),
    # achieved 8e-5 (r02g)
    assert gpu["sigma2"] == pytest.approx(g["sigma2"], rel=2e-4)


def test_concurrent_calls_on_two_threads_and_streams():
    # include/lsgcpd.h: calls on distinct streams are independent.  Two host threads, each with its own CUDA
    # stream, run registrations (graph capture, graph cache, per-device caches, the option store) at the same time;
    # every result equals the same call made alone.
    import threading
    import torch
    import paper_2103_15039_b200 as lsg
    import synth
    wls = synth.make_batch(2, 1500, seed=41)
    tgts = [lsg.prepare_target(to_dev(w.target), w.knn_k) for w in wls]
    srcs = [to_dev(w.source) for w in wls]
    alone = [lsg.register(t, x, 30, w=0.1) for t, x in zip(tgts, srcs)]
    out = [[None] * 4, [None] * 4]
    errs = []

    def worker(i):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for k in range(4):
                    out[i][k] = lsg.register(tgts[i], srcs[i], 30, w=0.1, stream=s)
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for i in range(2):
        for r in out[i]:
            assert r["iters"] == 30 and r["status"] == 0
            np.testing.assert_array_equal(r["R"], alone[i]["R"])
            np.testing.assert_array_equal(r["t"], alone[i]["t"])
            assert r["sigma2"] == alone[i]["sigma2"]


@pytest.mark.parametrize("name", ["rgbd", "lidar"])
def test_register_source_order_and_far_rule_do_not_change_the_result(name):
    # lsgcpd_register runs on a Morton-ordered copy of the source and lets far warps take the centred residual
    # (DESIGN §8 "far points"): against the given order with the rule off, only the FP summation order and the
    # residual's rounding differ, so the poses agree far inside the 1e-4 rad bar and σ² to the E step's FP32
    # rounding; with the same options the result is bit-for-bit repeatable
    import paper_2103_15039_b200 as lsg
    wl = workload(name)
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    X = to_dev(wl.source)
    out = {}
    for key, opts in (("plain", {"sort_source": 0, "far_rule": 0}), ("product", {}), ("again", {})):
        with lsg.options(**opts):
            out[key] = lsg.register(tgt, X, wl.iters, w=wl.w)
    a, b = out["plain"], out["product"]
    _close(b["R"], b["t"], a["R"], a["t"], float(np.linalg.norm(wl.target.max(0) - wl.target.min(0))), tol=1e-6)
    assert abs(b["sigma2"] / a["sigma2"] - 1.0) <= 1e-5, (b["sigma2"], a["sigma2"])
    assert np.array_equal(out["again"]["R"], b["R"]) and out["again"]["sigma2"] == b["sigma2"]


def test_register_workspace_holds_the_ordered_source_from_4096_points():
    # sources of >= 4,096 points are registered on a Morton-ordered copy kept in the workspace: the workspace
    # grows by at least the copy, its φ and the sort's keys and ids at that size (the query needs the device)
    import paper_2103_15039_b200 as lsg
    L = lsg.lib()
    below = L.lsgcpd_register_workspace_bytes(10000, 4095, 50)
    at = L.lsgcpd_register_workspace_bytes(10000, 4096, 50)
    assert below > 0 and at - below >= 4096 * (12 + 4 + 8 + 8 + 4 + 4)
