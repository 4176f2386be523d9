"""Target preparation parity (kNN, κ, n, α, V): GPU (lsgcpd_prepare_target) vs the FP64 oracle.
Tolerances: SURVEY §8(c).6 step 1 / DESIGN.md "Parity protocol"."""
import numpy as np
import pytest

import oracle
from tests.gpu_common import to_dev, workload

pytestmark = pytest.mark.gpu


def _check_stage(Y, ann, tg, rows, k):
    knn_g = ann["knn"].cpu().numpy()[rows]
    knn_o = tg["knn"]
    _, d2 = oracle.knn(Y, k + 1, queries=rows)
    same = np.all(knn_g == knn_o, axis=1)
    # a set may differ only at a near-tie between the k-th and (k+1)-th neighbour
    near_tie = (d2[:, k] - d2[:, k - 1]) <= 1e-6 * np.maximum(d2[:, k], 1e-300)
    assert np.all(same | near_tie), f"kNN mismatch at {np.flatnonzero(~(same | near_tie))[:10]}"
    ok = same
    kap_g = ann["kappa"].cpu().numpy()[rows][ok]
    np.testing.assert_allclose(kap_g, tg["kappa"][ok], atol=1e-6, rtol=0)
    a_g = ann["alpha"].cpu().numpy()[rows][ok]
    np.testing.assert_allclose(a_g, tg["alpha"][ok], rtol=1e-5, atol=1e-5)
    n_g = ann["normals"].cpu().numpy()[rows][ok].astype(np.float64)
    cosang = np.abs((n_g * tg["normals"][ok]).sum(1)) / np.linalg.norm(n_g, axis=1)
    ang = np.arccos(np.clip(cosang, -1, 1))
    ev = tg["evals"][ok]
    bound = 1e-6 * ev.sum(1) / np.maximum(ev[:, 1] - ev[:, 0], 1e-300) + 1e-6
    assert np.all((ang <= bound) | (tg["alpha"][ok] < 1e-6)), ang.max()


@pytest.mark.parametrize("name", ["tiny", "object"])
def test_prepare_parity_full(name):
    import paper_2103_15039_b200 as lsg
    wl = workload(name)
    Y = wl.target
    tgt, ann = lsg.prepare_target(to_dev(Y), wl.knn_k, annotations=True)
    tg = oracle.prepare_target(Y, wl.knn_k)
    _check_stage(Y, ann, tg, np.arange(wl.M), wl.knn_k)
    V, ext = oracle.working_volume(Y)
    assert tgt.volume == pytest.approx(V, rel=1e-12)
    assert tgt.extent == pytest.approx(ext, rel=1e-12)
    assert tgt.alpha_mean == pytest.approx(tg["alpha"].mean(), rel=1e-5)


@pytest.mark.parametrize("name", ["rgbd", "lidar", "scale"])
def test_prepare_parity_sampled(name):
    import paper_2103_15039_b200 as lsg
    wl = workload(name)
    Y = wl.target
    tgt, ann = lsg.prepare_target(to_dev(Y), wl.knn_k, annotations=True)
    rows = np.sort(np.random.default_rng(3).choice(wl.M, 400, replace=False))
    idx, _ = oracle.knn(Y, wl.knn_k, queries=rows)
    n, kappa, deg, evals = oracle.local_surface(Y, idx)
    tg = {"knn": idx, "kappa": kappa, "alpha": oracle.alpha_from_kappa(kappa), "normals": n, "evals": evals}
    _check_stage(Y, ann, tg, rows, wl.knn_k)
    ext = Y.astype(np.float64).max(0) - Y.astype(np.float64).min(0)
    assert tgt.volume == pytest.approx(np.prod(ext * 1.2), rel=1e-12)


def test_prepare_degenerate_inputs():
    import paper_2103_15039_b200 as lsg
    with pytest.raises(lsg.LsgcpdError, match="EDEGENERATE"):
        lsg.prepare_target(to_dev(np.ones((20, 3), np.float32)))
    # planar cloud: zero-extent axis floored at the mean nearest-neighbour spacing
    g = np.array([[x, y, 0.0] for x in np.arange(8) * 0.25 for y in np.arange(8) * 0.25], np.float32)
    tgt = lsg.prepare_target(to_dev(g), 10)
    V, _ = oracle.working_volume(g)
    assert tgt.volume == pytest.approx(V, rel=1e-6)
    # duplicates: coincident neighbourhoods are flagged, κ = 1/3, α = 0
    d = np.repeat(np.random.default_rng(1).uniform(-1, 1, (5, 3)), 12, axis=0).astype(np.float32)
    tgt, ann = lsg.prepare_target(to_dev(d), 10, annotations=True)
    assert tgt.n_degenerate == 60
    np.testing.assert_allclose(ann["alpha"].cpu().numpy(), 0.0, atol=1e-6)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.prepare_target(to_dev(np.zeros((2, 3), np.float32)))


@pytest.mark.parametrize("k", [3, 10, 32])
def test_prepare_knn_dense_cluster_with_far_outliers(k):
    # the three search paths of the kNN at once: a dense cluster (bulk grid: its box is far smaller than the
    # AABB the outliers inflate), points beside it (fine grid) and isolated outliers far out (one warp each on
    # the coarse grid); every point's k nearest against the brute-force oracle
    import paper_2103_15039_b200 as lsg
    rng = np.random.default_rng(41)
    dense = rng.normal(0.0, 0.01, (3000, 3))
    plane = np.c_[rng.uniform(-0.3, 0.3, (600, 2)), rng.normal(0.0, 1e-3, 600)]
    far = rng.uniform(-50.0, 50.0, (250, 3))
    Y = np.concatenate([dense, plane, far]).astype(np.float32)
    tgt, ann = lsg.prepare_target(to_dev(Y), k, annotations=True)
    tg = oracle.prepare_target(Y, k)
    _check_stage(Y, ann, tg, np.arange(Y.shape[0]), k)


def test_prepare_batch_equals_single_prepares():
    # lsgcpd_prepare_batch builds exactly (byte for byte) the targets B lsgcpd_prepare_target calls build,
    # for clouds of different sizes and kinds (one of them with far outliers: the bulk-grid path)
    import paper_2103_15039_b200 as lsg
    import synth
    clouds = [w.target for w in synth.make_batch(3, 900, seed=5, ragged=True)]
    rng = np.random.default_rng(2)
    clouds.append(np.concatenate([rng.normal(0, 0.02, (800, 3)), rng.uniform(-20, 20, (60, 3))]).astype(np.float32))
    clouds.append(workload("tiny").target)
    dev = [to_dev(c) for c in clouds]
    import torch
    junk = torch.full((256 << 20,), 0x5A, dtype=torch.uint8, device="cuda")   # the workspace is recycled, dirty
    del junk
    batch = lsg.prepare_batch(dev, 10)
    for c, tb in zip(dev, batch):
        ts = lsg.prepare_target(c, 10)
        assert tb.M == ts.M and tb.volume == ts.volume and tb.extent == ts.extent
        assert torch_equal(tb.buf, ts.buf)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.prepare_batch([to_dev(np.zeros((2, 3), np.float32))], 10)


def test_prepare_batch_several_waves_equal_single_prepares():
    # more targets than one wave holds: 70 small clouds (waves of 64 + 6), and a batch whose largest cloud (the
    # scale config's target) leaves room for only a few targets per wave; every target byte-identical to its
    # lsgcpd_prepare_target build, the workspace dirty
    import torch
    import paper_2103_15039_b200 as lsg
    import synth
    small = [to_dev(w.target) for w in synth.make_batch(70, 600, seed=9, ragged=True)]
    big = [to_dev(workload("scale").target)] + small[:7]
    for clouds, check in ((small, [0, 1, 63, 64, 65, 69]), (big, list(range(8)))):
        junk = torch.full((512 << 20,), 0xA5, dtype=torch.uint8, device="cuda")
        del junk
        batch = lsg.prepare_batch(clouds, 10)
        for b in check:
            ts = lsg.prepare_target(clouds[b], 10)
            assert torch_equal(batch[b].buf, ts.buf), f"target {b} of {len(clouds)}"


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


def test_prepare_batch_edge_cases():
    # B = 1 with the minimal cloud (M = k = 3), and a batch whose second cloud is degenerate: EDEGENERATE
    # naming that problem
    import paper_2103_15039_b200 as lsg
    tri = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0]], np.float32)
    (tb,) = lsg.prepare_batch([to_dev(tri)], 3)
    ts = lsg.prepare_target(to_dev(tri), 3)
    assert torch_equal(tb.buf, ts.buf)
    good = workload("tiny").target
    with pytest.raises(lsg.LsgcpdError, match="problem 1"):
        lsg.prepare_batch([to_dev(good), to_dev(np.ones((50, 3), np.float32))], 10)
    # a degenerate cloud in the second wave (64 targets per wave): refused before any wave runs, named
    clouds = [to_dev(good)] * 69 + [to_dev(np.ones((50, 3), np.float32))]
    with pytest.raises(lsg.LsgcpdError, match="problem 69"):
        lsg.prepare_batch(clouds, 10)
