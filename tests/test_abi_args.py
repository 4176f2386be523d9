"""Argument validation at the C ABI, on the CPU: empty, out-of-range and non-finite arguments are refused with
LSGCPD_EINVAL and a message before any device work (include/lsgcpd.h "Errors"), so these run without a GPU.
The fake device pointers below are never dereferenced: every call fails validation first."""
import ctypes

import numpy as np
import pytest

EINVAL = -1
FAKE = 0x10000          # 16-byte aligned, never dereferenced


@pytest.fixture(scope="module")
def L():
    from paper_2103_15039_b200 import build
    build.build()
    import paper_2103_15039_b200 as pkg
    return pkg.lib()


def _pose():
    R = (ctypes.c_double * 9)(1, 0, 0, 0, 1, 0, 0, 0, 1)
    t = (ctypes.c_double * 3)(0, 0, 0)
    return ctypes.cast(R, ctypes.POINTER(ctypes.c_double)), ctypes.cast(t, ctypes.POINTER(ctypes.c_double))


def _estep(L, M, N, s2=1e-3, w=0.1, V=1.0, R=None, t=None):
    R0, t0 = _pose()
    return L.lsgcpd_estep(FAKE, M, FAKE, N, R or R0, t or t0, s2, w, V, 1, FAKE, FAKE, 1 << 40, None)


def _err(L):
    return L.lsgcpd_last_error().decode()


@pytest.mark.parametrize("M,N", [(0, 10), (10, 0), (0, 0), (-5, 10), (1 << 30, 10), (10, 1 << 34)])
def test_estep_empty_and_out_of_range_sizes(L, M, N):
    assert _estep(L, M, N) == EINVAL
    assert "out of range" in _err(L)


@pytest.mark.parametrize("kw,msg", [(dict(s2=0.0), "sigma2"), (dict(s2=float("nan")), "sigma2"),
                                    (dict(w=1.0), "w must"), (dict(w=-0.1), "w must"), (dict(V=0.0), "volume"),
                                    (dict(V=float("inf")), "volume")])
def test_estep_bad_scalars(L, kw, msg):
    assert _estep(L, 100, 100, **kw) == EINVAL
    assert msg in _err(L)


def test_estep_bad_pose_and_pointers(L):
    Rb = (ctypes.c_double * 9)(2, 0, 0, 0, 1, 0, 0, 0, 1)                 # not a rotation
    assert _estep(L, 100, 100, R=ctypes.cast(Rb, ctypes.POINTER(ctypes.c_double))) == EINVAL
    Rr = (ctypes.c_double * 9)(1, 0, 0, 0, -1, 0, 0, 0, -1)               # det +1 reflection pair: a rotation
    tn = (ctypes.c_double * 3)(np.nan, 0, 0)
    assert _estep(L, 100, 100, R=ctypes.cast(Rr, ctypes.POINTER(ctypes.c_double)),
                  t=ctypes.cast(tn, ctypes.POINTER(ctypes.c_double))) == EINVAL
    assert "t must be finite" in _err(L)
    R0, t0 = _pose()
    assert L.lsgcpd_estep(None, 10, FAKE, 10, R0, t0, 1e-3, 0.1, 1.0, 1, FAKE, FAKE, 1 << 40, None) == EINVAL
    assert L.lsgcpd_estep(FAKE + 4, 10, FAKE, 10, R0, t0, 1e-3, 0.1, 1.0, 1, FAKE, FAKE, 1 << 40, None) == EINVAL
    assert "aligned" in _err(L)


def test_workspace_queries_refuse_empty_sizes(L):
    assert L.lsgcpd_estep_workspace_bytes(0, 10) == 0
    assert L.lsgcpd_estep_workspace_bytes(10, 0) == 0
    assert L.lsgcpd_register_workspace_bytes(10, 0, 5) == 0
    assert L.lsgcpd_register_workspace_bytes(10, 10, -1) == 0
    assert L.lsgcpd_select_workspace_bytes(0) == 0
    assert L.lsgcpd_target_prior_workspace_bytes(0) == 0
    assert L.lsgcpd_prepare_workspace_bytes(-1, 10) == 0


def test_prepare_register_and_model_extensions_refuse_bad_arguments(L):
    import paper_2103_15039_b200 as pkg
    info = pkg.TargetInfo()
    # prepare: M < 3, k out of range
    assert L.lsgcpd_prepare_target(FAKE, 2, None, FAKE, FAKE, 1 << 40, ctypes.byref(info), None, None) == EINVAL
    pp = pkg.PrepParams()
    L.lsgcpd_prep_params_default(ctypes.byref(pp))
    pp.knn_k = 40
    assert L.lsgcpd_prepare_target(FAKE, 100, ctypes.byref(pp), FAKE, FAKE, 1 << 40, ctypes.byref(info), None,
                                   None) == EINVAL
    # register: empty local shard, w out of range, eta ≥ 1, unknown group
    ep = pkg.EmParams()
    L.lsgcpd_em_params_default(ctypes.byref(ep))
    Ro = (ctypes.c_double * 9)()
    to = (ctypes.c_double * 3)()
    s2 = ctypes.c_double()
    it = ctypes.c_int()
    dp = ctypes.POINTER(ctypes.c_double)

    def reg(N, p):
        return L.lsgcpd_register(FAKE, 100, 0.0, FAKE, N, ctypes.byref(p), None, None, ctypes.cast(Ro, dp),
                                 ctypes.cast(to, dp), ctypes.byref(s2), ctypes.byref(it), None, None, None, FAKE,
                                 1 << 40, None)
    assert reg(0, ep) == EINVAL
    for field, val in (("w", 1.0), ("eta", 1.0), ("group", 2), ("max_iters", -1), ("newton_max", 5000)):
        bad = pkg.EmParams()
        L.lsgcpd_em_params_default(ctypes.byref(bad))
        setattr(bad, field, val)
        assert reg(100, bad) == EINVAL, field
    # batch: no problems
    assert L.lsgcpd_register_batch(None, 0, None, ctypes.cast(Ro, dp), ctypes.cast(to, dp), ctypes.cast(to, dp),
                                   ctypes.byref(it), ctypes.byref(it), FAKE, 1 << 40, None) == EINVAL
    # truncation and the depth error model: empty input, non-finite threshold, a zero error model
    n_out = ctypes.c_int64()
    assert L.lsgcpd_select_confident(FAKE, FAKE, 0, 0.5, FAKE, FAKE, ctypes.byref(n_out), FAKE, 1 << 40,
                                     None) == EINVAL
    assert L.lsgcpd_select_confident(FAKE, FAKE, 10, float("nan"), FAKE, FAKE, ctypes.byref(n_out), FAKE, 1 << 40,
                                     None) == EINVAL
    assert L.lsgcpd_depth_confidence(FAKE, 0, 0.0, 0.002, 0.4, FAKE, None) == EINVAL
    assert L.lsgcpd_depth_confidence(FAKE, 10, 0.0, 0.0, 0.4, FAKE, None) == EINVAL


def test_prepare_batch_workspace_is_bounded(L):
    # waves of up to 64 targets within ~512 MB of job regions: 550 paper-scale clouds stay under 1 GiB, and a
    # batch holding a 2^29-point cloud gets one target per wave (no int overflow in the wave's sort offsets)
    M = (ctypes.c_int64 * 550)(*([3500] * 550))
    ws = L.lsgcpd_prepare_batch_workspace_bytes(M, 550, 10)
    assert 0 < ws < (1 << 30)
    M1 = (ctypes.c_int64 * 1)(3500)
    assert L.lsgcpd_prepare_batch_workspace_bytes(M1, 1, 10) < ws   # one target: one job region
    big = (ctypes.c_int64 * 2)(1 << 29, 5)
    assert L.lsgcpd_prepare_batch_workspace_bytes(big, 2, 10) >= L.lsgcpd_prepare_workspace_bytes(1 << 29, 10)


def test_prepare_batch_refuses_bad_arguments(L):
    M = (ctypes.c_int64 * 2)(100, 2)
    assert L.lsgcpd_prepare_batch_workspace_bytes(M, 2, 10) == 0          # a cloud with M < 3
    M_ok = (ctypes.c_int64 * 2)(100, 50)
    assert L.lsgcpd_prepare_batch_workspace_bytes(M_ok, 0, 10) == 0       # B < 1
    assert L.lsgcpd_prepare_batch_workspace_bytes(M_ok, 2, 10) > 0
    ptrs = (ctypes.c_void_p * 2)(FAKE, FAKE)
    assert L.lsgcpd_prepare_batch(ptrs, M, 2, None, ptrs, FAKE, 1 << 40, None, None) == EINVAL
    assert "problem 1" in _err(L)
    assert L.lsgcpd_prepare_batch(ptrs, M_ok, 0, None, ptrs, FAKE, 1 << 40, None, None) == EINVAL
    unaligned = (ctypes.c_void_p * 2)(FAKE, FAKE + 4)
    assert L.lsgcpd_prepare_batch(ptrs, M_ok, 2, None, unaligned, FAKE, 1 << 40, None, None) == EINVAL


def test_options_set_get_and_refusals(L):
    import paper_2103_15039_b200 as lsg
    old = lsg.get_option("tile_gate")
    with lsg.options(tile_gate=7.5, tc=0, estep_variant=1):
        assert lsg.get_option("tile_gate") == 7.5
        assert lsg.get_option("tc") == 0 and lsg.get_option("estep_variant") == 1
    assert lsg.get_option("tile_gate") == old and lsg.get_option("tc") == 2
    assert L.lsgcpd_set_option(b"no_such_option", 1.0) == EINVAL and "unknown option" in _err(L)
    assert L.lsgcpd_set_option(b"tc", 3.0) == EINVAL
    assert L.lsgcpd_set_option(b"estep_variant", 5.0) == EINVAL
    assert L.lsgcpd_set_option(b"tile_gate", float("nan")) == EINVAL
    assert L.lsgcpd_set_option(None, 1.0) == EINVAL


@pytest.mark.parametrize("G", [0, -1, 17])
def test_register_shards_shard_count_refused(L, G):
    import paper_2103_15039_b200 as lsg
    R0, t0 = _pose()
    ptrs = (ctypes.c_void_p * 17)(*([FAKE] * 17))
    Ns = (ctypes.c_int64 * 17)(*([100] * 17))
    R = np.zeros(9 * 17)
    t = np.zeros(3 * 17)
    s2 = np.zeros(17)
    it = (ctypes.c_int * 17)()
    dp = ctypes.POINTER(ctypes.c_double)
    rc = L.lsgcpd_register_shards(FAKE, 100, 0.0, ptrs, Ns, G, None, R0, t0, R.ctypes.data_as(dp),
                                  t.ctypes.data_as(dp), s2.ctypes.data_as(dp), it, FAKE, 1 << 20, None)
    assert rc == EINVAL and "out of range" in _err(L)

