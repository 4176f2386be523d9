"""Registration parity at the BASELINE configs' full sizes (rgbd, lidar, scale), where a full FP64 oracle
registration takes 0.5-12 h: teacher forcing.  At EM states k taken from the GPU's
own trajectory (lsgcpd_register stopped after k iterations):
  * E step: the GPU record at (R_k, t_k, σ²_k) vs the oracle's Eq. 5 record on sampled source points
    (every target), tolerance 2e-5 of scale (tests/parity.py);
  * M step: the oracle's damped Newton + σ² update (oracle/mstep.py) run on the GPU's full
    record must land where the GPU's iteration k+1 landed: R within 1e-4 rad, t within 1e-4·extent
    (the north-star bar), σ² within 1e-6 relative.
Each EM step of the GPU trajectory is then an oracle step within tolerance, for the whole run.
Also: the NCCL all-reduce path of lsgcpd_register with a one-rank communicator equals the no-comm path."""
import numpy as np
import pytest

import oracle
from oracle import se3
from tests.gpu_common import to_dev, workload
from tests.parity import assert_record_parity, transformed

pytestmark = pytest.mark.gpu


def _states(iters):
    return sorted({0, 1, iters // 2, iters - 1})


@pytest.mark.parametrize("name", ["rgbd", "lidar", "scale"])
def test_register_teacher_forced_full_scale(name):
    import paper_2103_15039_b200 as lsg
    wl = workload(name)
    tgt, ann = lsg.prepare_target(to_dev(wl.target), wl.knn_k, annotations=True)
    n64 = ann["normals"].cpu().numpy().astype(np.float64)
    a64 = ann["alpha"].cpu().numpy().astype(np.float64)
    X = to_dev(wl.source)
    iters = wl.iters
    reg = lsg.Registrar(tgt, X, iters)
    rng = np.random.default_rng(17)
    idx = np.sort(rng.choice(wl.N, 1024, replace=False))
    floor = 1e-12 * tgt.extent ** 2
    first = lsg.Registrar(tgt, X, 1)(w=wl.w, traces=True)
    for k in _states(iters):
        if k == 0:
            R, t, s2 = np.eye(3), np.zeros(3), float(first["sigma2_trace"][0])
        else:
            st = lsg.Registrar(tgt, X, k)(w=wl.w)
            assert st["iters"] == k and st["status"] == 0
            R, t, s2 = st["R"], st["t"], st["sigma2"]
        nxt = first if k == 0 else lsg.Registrar(tgt, X, k + 1)(w=wl.w)
        rec = lsg.estep(tgt, X, R, t, s2, wl.w, tgt.volume).cpu().numpy()
        ora = oracle.estep(wl.target, n64, a64, wl.source[idx], R, t, s2, wl.w, tgt.volume)
        assert_record_parity(rec[idx], ora, wl.target, a64, what=f"{name} E step at state {k}",
                             Xh=transformed(wl.source[idx], R, t), s2=s2)
        R1, t1, s21, _ = oracle.mstep(wl.source, rec, R, t, s2, tgt.extent, 10, floor)
        ang = se3.rotation_angle(np.asarray(nxt["R"]).T @ R1)
        dt = np.linalg.norm(np.asarray(nxt["t"]) - t1)
        assert ang <= 1e-4, f"{name} M step {k}: rotation differs by {ang:.2e} rad"
        assert dt <= 1e-4 * tgt.extent, f"{name} M step {k}: translation differs by {dt:.2e}"
        assert abs(nxt["sigma2"] - s21) <= 1e-6 * s21, (name, k, nxt["sigma2"], s21)
    del reg


@pytest.mark.parametrize("no_fuse", ["0", "1"])
def test_register_with_one_rank_nccl_comm_equals_no_comm(no_fuse):
    # the communicator path (ncclAllReduce of the 75 moments per iteration) with world size 1, after the fused
    # merge + moments kernel (N ≤ 2^17) and after the separate merge / moments kernels (the N > 2^17 path)
    import paper_2103_15039_b200 as lsg
    with lsg.options(no_fuse=int(no_fuse)):
        _one_rank_comm(lsg)


def _one_rank_comm(lsg):
    wl = workload("object")
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    X = to_dev(wl.source)
    reg = lsg.Registrar(tgt, X, 20)
    plain = reg(w=wl.w, traces=True)
    comm = lsg.Comm(0, 1)
    try:
        viac = reg(w=wl.w, traces=True, comm=comm)
    finally:
        comm.close()
    assert viac["iters"] == plain["iters"] == 20
    assert np.array_equal(viac["R"], plain["R"]) and np.array_equal(viac["t"], plain["t"])
    assert viac["sigma2"] == plain["sigma2"]
    np.testing.assert_array_equal(viac["nll"], plain["nll"])


def test_estep_indexing_beyond_2_31_record_floats():
    # maximum-size edge case: N·16 > 2^31 record floats (and a partial buffer twice that), so every source
    # offset past point 2^27 needs 64-bit indexing in the pair kernels, the merge and the record store.
    # Source: the tiny workload tiled with a per-copy shift, built on the device from the seeded input by the
    # same float32 formula the host repeats for the sampled rows.
    import torch
    import paper_2103_15039_b200 as lsg
    from tests.gpu_common import oracle_target32
    wl, n32, a32, V, ext = oracle_target32("tiny")
    tgt = lsg.pack_target(to_dev(wl.target), to_dev(n32), to_dev(a32))
    N = (1 << 27) + 77
    base = torch.from_numpy(wl.source).cuda()
    k = torch.arange(N, device="cuda")
    X = base[k % wl.N] + ((k // wl.N).to(torch.float32) * np.float32(1e-7))[:, None]
    del k
    R, t = wl.R_expected, wl.t_expected
    s2 = 1e-3
    rec = lsg.estep(tgt, X, R, t, s2, wl.w, V)
    rng = np.random.default_rng(29)
    idx = np.unique(np.concatenate([rng.choice(N, 40, replace=False), np.arange(N - 8, N),
                                    np.arange((1 << 27) - 4, (1 << 27) + 4)]))
    sub = rec[torch.from_numpy(idx).cuda()].cpu().numpy()
    del rec, X
    torch.cuda.empty_cache()
    xs = wl.source[idx % wl.N] + ((idx // wl.N).astype(np.float32) * np.float32(1e-7))[:, None]
    ora = oracle.estep(wl.target, n32.astype(np.float64), a32.astype(np.float64), xs.astype(np.float32), R, t, s2,
                       wl.w, V)
    assert_record_parity(sub, ora, wl.target, a32, what="N = 2^27 + 77 sampled", Xh=transformed(xs, R, t), s2=s2)


def test_estep_targets_beyond_2_31_bytes():
    # maximum-size edge case on the target side: M = 2^24 + 5 targets (2.7 GB of prepared target, tile offsets
    # past 2^31 bytes), every one of them within reach of every source point (the tiny target tiled with a
    # 1e-7 shift per copy), so the sums run over all 16.8 M targets, against the oracle on sampled points.
    import paper_2103_15039_b200 as lsg
    from tests.gpu_common import oracle_target32
    wl, n32, a32, _, _ = oracle_target32("tiny")
    M = (1 << 24) + 5
    k = np.arange(M)
    Y = wl.target[k % wl.M] + ((k // wl.M).astype(np.float32) * np.float32(1e-7))[:, None]
    nY, aY = n32[k % wl.M], a32[k % wl.M]
    del k
    V, _ = oracle.working_volume(Y)
    tgt = lsg.pack_target(to_dev(Y), to_dev(nY), to_dev(aY))
    X = wl.source[:64]
    R, t = wl.R_expected, wl.t_expected
    for s2 in (1e-3, 1e-5):
        rec = lsg.estep(tgt, to_dev(X), R, t, s2, wl.w, V).cpu().numpy()
        ora = oracle.estep(Y, nY.astype(np.float64), aY.astype(np.float64), X, R, t, s2, wl.w, V)
        assert_record_parity(rec, ora, Y, aY, what=f"M = 2^24 + 5, s2={s2}", Xh=transformed(X, R, t), s2=s2)


@pytest.mark.parametrize("comm", [False, True])
def test_register_without_graph_equals_graph(comm):
    # the plain-launch EM loop (option no_graph; the path of a communicator with more than one rank, whose
    # iterations are not captured) gives the captured graph's result bit for bit, with and without a one-rank
    # NCCL communicator
    import paper_2103_15039_b200 as lsg
    wl = workload("object")
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    X = to_dev(wl.source)
    reg = lsg.Registrar(tgt, X, 20)
    c = lsg.Comm(0, 1) if comm else None
    try:
        graph = reg(w=wl.w, traces=True, comm=c)
        with lsg.options(no_graph=1):
            plain = reg(w=wl.w, traces=True, comm=c)
    finally:
        if c is not None:
            c.close()
    assert plain["iters"] == graph["iters"] == 20
    assert np.array_equal(plain["R"], graph["R"]) and np.array_equal(plain["t"], graph["t"])
    assert plain["sigma2"] == graph["sigma2"]
    np.testing.assert_array_equal(plain["nll"], graph["nll"])
