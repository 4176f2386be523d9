"""Multi-rank host path on CPU (gloo, world size 2): sharding, the 128-byte communicator-id broadcast, and
the property the sharded GPU registration relies on — EM over source shards whose M-step sums are
all-reduced equals EM over the whole source (checked with the FP64 oracle on each rank)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2103_15039_b200.dist import shard_range


def test_shard_range_partitions():
    for n in (0, 1, 7, 1000, 524288):
        for world in (1, 2, 3, 4, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [hi - lo for lo, hi in parts]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _sharded_newton(stats, extent, newton_max, allreduce):
    """Damped Newton of oracle/mstep.py with every per-point sum all-reduced across ranks."""
    from oracle import se3
    R, t = stats.R_E.copy(), stats.t_E.copy()
    q_cur = 0.0
    for _ in range(newton_max):
        g, H = stats.grad_hess(R, t)
        gH = allreduce(np.concatenate([g, H.ravel()]))
        g, H = gH[:6], gH[6:].reshape(6, 6)
        tr = abs(np.trace(H)) / 6.0
        mu, accepted, converged = 0.0, False, False
        for _ in range(20):
            try:
                L = np.linalg.cholesky(H + mu * np.eye(6))
            except np.linalg.LinAlgError:
                mu = max(10 * mu, 1e-6 * tr)
                continue
            d = -np.linalg.solve(L.T, np.linalg.solve(L, g))
            if np.linalg.norm(d[:3]) < 1e-10 and np.linalg.norm(d[3:]) < 1e-10 * extent:
                converged = True
                break
            Rn, tn = se3.compose(R, t, *se3.exp(d))
            qn = float(allreduce(np.array([stats.q_rel(Rn, tn)]))[0])
            if qn < q_cur:
                R, t, q_cur, accepted = Rn, tn, qn, True
                break
            mu = max(10 * mu, 1e-6 * tr)
        if converged or not accepted:
            break
    return R, t, q_cur


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    import synth
    from paper_2103_15039_b200.dist import broadcast_bytes
    # the communicator id travels as 128 bytes from rank 0
    blob = broadcast_bytes(bytes(range(128)) if rank == 0 else b"", 0)
    assert blob == bytes(range(128))

    def allreduce(v):
        t = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64))
        dist.all_reduce(t)
        return t.numpy()

    wl = synth.make("tiny")
    tg = oracle.prepare_target(wl.target, wl.knn_k)
    V, ext = oracle.working_volume(wl.target)
    lo, hi = shard_range(wl.N, rank, world)
    X = wl.source[lo:hi].astype(np.float64)
    # σ²₀ from all-reduced centred sums (lsgcpd_register's σ²₀ all-reduce)
    yb = wl.target.astype(np.float64).mean(0)
    sx, n = allreduce(np.array([((X - yb) ** 2).sum(), len(X)]))
    s2 = (wl.M * sx + n * ((wl.target - yb) ** 2).sum()) / (3 * wl.M * n)
    R, t = np.eye(3), np.zeros(3)
    for _ in range(15):
        rec = oracle.estep(tg["Y"], tg["normals"], tg["alpha"], X, R, t, s2, wl.w, V, nthreads=1)
        st = oracle.PointStats(X, rec, R, t, s2)
        R, t, q = _sharded_newton(st, ext, 10, allreduce)
        sig2D, sumP = allreduce(np.array([st.sig2D.sum(), st.P.sum()]))
        s2 = max(1e-12 * ext * ext, (sig2D + q) / (3 * sumP))
    out[rank] = np.concatenate([R.ravel(), t, [s2]])
    dist.destroy_process_group()


def test_two_rank_sharded_em_equals_single_process():
    import oracle
    import synth
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    a, b = out[0], out[1]
    np.testing.assert_array_equal(a, b)                       # identical pose on every rank
    wl = synth.make("tiny")
    tg = oracle.prepare_target(wl.target, wl.knn_k)
    V, ext = oracle.working_volume(wl.target)
    ref = oracle.register(tg, wl.source, wl.w, 15, V, ext)
    np.testing.assert_allclose(a[:9], ref["R"].ravel(), atol=1e-10)
    np.testing.assert_allclose(a[9:12], ref["t"], atol=1e-10)
    assert a[12] == pytest.approx(ref["sigma2"], rel=1e-9)


def _subgroup_worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2103_15039_b200.dist import broadcast_bytes
    grp = dist.new_group([1, 2])   # group ranks 0, 1 = global ranks 1, 2
    if rank in (1, 2):
        # `src` is the GROUP rank: group rank 0 is global rank 1, which holds the id
        blob = broadcast_bytes(b"id-from-global-1" if rank == 1 else b"", 0, grp)
        out[rank] = blob
    dist.barrier()
    dist.destroy_process_group()


def test_broadcast_bytes_in_a_subgroup_uses_group_ranks():
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_subgroup_worker, args=(3, port, out), nprocs=3, join=True)
    assert out[1] == b"id-from-global-1" and out[2] == b"id-from-global-1"
