"""B200-native LSG-CPD (arXiv 2103.15039): Python binding of liblsgcpd.so.

The binding only marshals arguments: every step of the path (target preparation, E step, moments,
Newton M step, σ² update, EM loop) runs in the library's sm_100a kernels.  PyTorch provides device
memory, streams and process groups.  There is NO CPU fallback: if the shared library cannot be
loaded, importing the binding's functions raises.

Low-level names mirror the C ABI (include/lsgcpd.h): lsgcpd_estep, lsgcpd_register, ...
High-level helpers (prepare_target, pack_target, estep, register, Comm) wrap them for torch tensors.
"""
from __future__ import annotations

import ctypes
import os
import threading
from dataclasses import dataclass
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LSGCPD_LIB") or os.path.join(_HERE, "liblsgcpd.so")

REC = 16
REC_P, REC_PY, REC_A, REC_B, REC_D, REC_LNP, REC_POUT = 0, 1, 4, 10, 13, 14, 15
ERRORS = {0: "OK", -1: "EINVAL", -2: "EDEGENERATE", -3: "ECUDA", -4: "ENCCL", -5: "ENOMASS"}


class LsgcpdError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class PrepParams(ctypes.Structure):
    _fields_ = [("alpha_max", ctypes.c_float), ("lambda_", ctypes.c_float), ("knn_k", ctypes.c_int),
                ("volume_margin", ctypes.c_double)]


class TargetInfo(ctypes.Structure):
    _fields_ = [("volume", ctypes.c_double), ("extent", ctypes.c_double), ("aabb_lo", ctypes.c_double * 3),
                ("aabb_hi", ctypes.c_double * 3), ("alpha_mean", ctypes.c_double), ("n_degenerate", ctypes.c_int64)]


class Annotations(ctypes.Structure):
    _fields_ = [("d_normals", ctypes.c_void_p), ("d_kappa", ctypes.c_void_p), ("d_alpha", ctypes.c_void_p),
                ("d_knn", ctypes.c_void_p)]


class EmParams(ctypes.Structure):
    _fields_ = [("w", ctypes.c_double), ("max_iters", ctypes.c_int), ("newton_max", ctypes.c_int),
                ("consistent_normalizer", ctypes.c_int), ("sigma2_init", ctypes.c_double),
                ("sigma2_floor_rel", ctypes.c_double), ("tol", ctypes.c_double), ("eta", ctypes.c_double),
                ("d_src_conf", ctypes.c_void_p), ("group", ctypes.c_int)]


class Problem(ctypes.Structure):
    _fields_ = [("d_target", ctypes.c_void_p), ("M", ctypes.c_int64), ("d_src", ctypes.c_void_p), ("N", ctypes.c_int64),
                ("d_src_conf", ctypes.c_void_p), ("volume", ctypes.c_double), ("R0", ctypes.c_double * 9),
                ("t0", ctypes.c_double * 3)]


_lock = threading.Lock()
_lib = None

_vp, _i64, _i32, _d, _sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_size_t
_dp = ctypes.POINTER(ctypes.c_double)
_SIGS = {
    "lsgcpd_version": ([], _i32),
    "lsgcpd_last_error": ([], ctypes.c_char_p),
    "lsgcpd_prep_params_default": ([ctypes.POINTER(PrepParams)], None),
    "lsgcpd_em_params_default": ([ctypes.POINTER(EmParams)], None),
    "lsgcpd_target_bytes": ([_i64], _sz),
    "lsgcpd_prepare_workspace_bytes": ([_i64, _i32], _sz),
    "lsgcpd_prepare_target": ([_vp, _i64, ctypes.POINTER(PrepParams), _vp, _vp, _sz, ctypes.POINTER(TargetInfo),
                               ctypes.POINTER(Annotations), _vp], _i32),
    "lsgcpd_prepare_batch_workspace_bytes": ([ctypes.POINTER(ctypes.c_int64), _i32, _i32], _sz),
    "lsgcpd_prepare_batch": ([ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64), _i32,
                              ctypes.POINTER(PrepParams), ctypes.POINTER(ctypes.c_void_p), _vp, _sz,
                              ctypes.POINTER(TargetInfo), _vp], _i32),
    "lsgcpd_pack_workspace_bytes": ([_i64], _sz),
    "lsgcpd_pack_target": ([_vp, _vp, _vp, _i64, _d, _vp, _vp, _sz, ctypes.POINTER(TargetInfo), _vp], _i32),
    "lsgcpd_estep_workspace_bytes": ([_i64, _i64], _sz),
    "lsgcpd_estep": ([_vp, _i64, _vp, _i64, _dp, _dp, _d, _d, _d, _i32, _vp, _vp, _sz, _vp], _i32),
    "lsgcpd_estep_ex": ([_vp, _i64, _vp, _i64, _dp, _dp, _d, ctypes.POINTER(EmParams), _d, _vp, _vp, _sz, _vp], _i32),
    "lsgcpd_target_prior_workspace_bytes": ([_i64], _sz),
    "lsgcpd_target_set_prior": ([_vp, _i64, _vp, _vp, _sz, _dp, _vp], _i32),
    "lsgcpd_select_workspace_bytes": ([_i64], _sz),
    "lsgcpd_select_confident": ([_vp, _vp, _i64, ctypes.c_float, _vp, _vp, ctypes.POINTER(ctypes.c_int64), _vp, _sz,
                                 _vp], _i32),
    "lsgcpd_depth_confidence": ([_vp, _i64, _d, _d, _d, _vp, _vp], _i32),
    "lsgcpd_register_batch_workspace_bytes": ([ctypes.POINTER(Problem), _i32, _i32], _sz),
    "lsgcpd_register_batch": ([ctypes.POINTER(Problem), _i32, ctypes.POINTER(EmParams), _dp, _dp, _dp,
                               ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int), _vp, _sz, _vp], _i32),
    "lsgcpd_comm_unique_id": ([_vp], _i32),
    "lsgcpd_comm_init": ([_i32, _i32, _vp, ctypes.POINTER(ctypes.c_void_p)], _i32),
    "lsgcpd_comm_destroy": ([_vp], _i32),
    "lsgcpd_register_workspace_bytes": ([_i64, _i64, _i32], _sz),
    "lsgcpd_register": ([_vp, _i64, _d, _vp, _i64, ctypes.POINTER(EmParams), _dp, _dp, _dp, _dp, _dp,
                         ctypes.POINTER(ctypes.c_int), _dp, _dp, _vp, _vp, _sz, _vp], _i32),
    "lsgcpd_register_shards": ([_vp, _i64, _d, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_int64), _i32,
                                ctypes.POINTER(EmParams), _dp, _dp, _dp, _dp, _dp, ctypes.POINTER(ctypes.c_int), _vp,
                                _sz, _vp], _i32),
    "lsgcpd_set_option": ([ctypes.c_char_p, _d], _i32),
    "lsgcpd_get_option": ([ctypes.c_char_p, _dp], _i32),
}


def lib():
    """Load liblsgcpd.so (raises if it is missing — there is no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2103_15039_b200.build` "
                                  "(the CUDA extension is required; there is no CPU fallback)")
            L = ctypes.CDLL(LIB_PATH)
            for name, (args, res) in _SIGS.items():
                f = getattr(L, name)
                f.argtypes = args
                f.restype = res
            _lib = L
    return _lib


def _check(rc: int):
    if rc != 0:
        raise LsgcpdError(rc, lib().lsgcpd_last_error().decode(errors="replace"))


def _darr(a, n):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(n))
    return a, a.ctypes.data_as(_dp)


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _need_cuda_f32(t, name, cols=None):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA torch tensor")
    if t.dtype != torch.float32 or not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous float32")
    if cols is not None and (t.dim() != 2 or t.shape[1] != cols):
        raise ValueError(f"{name} must have shape [n, {cols}]")
    return t


# ---------------------------------------------------------------------------------------------
# high-level helpers (torch tensors in, torch tensors / numpy out)
# ---------------------------------------------------------------------------------------------

@dataclass
class Target:
    buf: "object"          # torch uint8 CUDA tensor holding the prepared target
    M: int
    volume: float
    extent: float
    alpha_mean: float
    n_degenerate: int
    aabb_lo: tuple
    aabb_hi: tuple


def _alloc_bytes(n, device):
    import torch
    return torch.empty(max(int(n), 16), dtype=torch.uint8, device=device)


def _target_from_info(buf, M, info):
    return Target(buf, M, info.volume, info.extent, info.alpha_mean, int(info.n_degenerate),
                  tuple(info.aabb_lo), tuple(info.aabb_hi))


def prepare_target(xyz, knn_k: int = 10, alpha_max: float = 50.0, lam: float = 0.5, volume_margin: float = 0.1,
                   annotations: bool = False, stream=None):
    """lsgcpd_prepare_target on a [M,3] float32 CUDA tensor.  Returns Target (and the annotations
    dict {normals, kappa, alpha, knn} when requested)."""
    import torch
    _need_cuda_f32(xyz, "xyz", 3)
    M = int(xyz.shape[0])
    L = lib()
    buf = _alloc_bytes(L.lsgcpd_target_bytes(M), xyz.device)
    ws = _alloc_bytes(L.lsgcpd_prepare_workspace_bytes(M, knn_k), xyz.device)
    p = PrepParams(alpha_max, lam, knn_k, volume_margin)
    info = TargetInfo()
    ann = None
    ann_t = None
    if annotations:
        ann_t = {"normals": torch.empty((M, 3), dtype=torch.float32, device=xyz.device),
                 "kappa": torch.empty(M, dtype=torch.float32, device=xyz.device),
                 "alpha": torch.empty(M, dtype=torch.float32, device=xyz.device),
                 "knn": torch.empty((M, knn_k), dtype=torch.int32, device=xyz.device)}
        ann = Annotations(ann_t["normals"].data_ptr(), ann_t["kappa"].data_ptr(), ann_t["alpha"].data_ptr(),
                          ann_t["knn"].data_ptr())
    _check(L.lsgcpd_prepare_target(xyz.data_ptr(), M, ctypes.byref(p), buf.data_ptr(), ws.data_ptr(), ws.numel(),
                                   ctypes.byref(info), ctypes.byref(ann) if ann is not None else None,
                                   _stream_ptr(stream)))
    tgt = _target_from_info(buf, M, info)
    return (tgt, ann_t) if annotations else tgt


def prepare_batch(clouds, knn_k: int = 10, alpha_max: float = 50.0, lam: float = 0.5, volume_margin: float = 0.1,
                  stream=None):
    """lsgcpd_prepare_batch: one Target per [M_b,3] float32 CUDA tensor, all prepared in one call."""
    B = len(clouds)
    if B < 1:
        raise ValueError("need at least one cloud")
    for c in clouds:
        _need_cuda_f32(c, "cloud", 3)
    L = lib()
    Ms = (ctypes.c_int64 * B)(*[int(c.shape[0]) for c in clouds])
    bufs = [_alloc_bytes(L.lsgcpd_target_bytes(int(c.shape[0])), clouds[0].device) for c in clouds]
    xs = (ctypes.c_void_p * B)(*[c.data_ptr() for c in clouds])
    ts = (ctypes.c_void_p * B)(*[b.data_ptr() for b in bufs])
    nbytes = L.lsgcpd_prepare_batch_workspace_bytes(Ms, B, knn_k)
    if nbytes == 0:
        raise LsgcpdError(-1, "invalid batch of clouds")
    ws = _alloc_bytes(nbytes, clouds[0].device)
    p = PrepParams(alpha_max, lam, knn_k, volume_margin)
    infos = (TargetInfo * B)()
    _check(L.lsgcpd_prepare_batch(xs, Ms, B, ctypes.byref(p), ts, ws.data_ptr(), ws.numel(), infos,
                                  _stream_ptr(stream)))
    return [_target_from_info(bufs[b], int(Ms[b]), infos[b]) for b in range(B)]


def pack_target(xyz, normals, alpha, volume_margin: float = 0.1, stream=None) -> Target:
    """lsgcpd_pack_target: target model from given normals [M,3] and α [M] (float32 CUDA tensors)."""
    _need_cuda_f32(xyz, "xyz", 3)
    _need_cuda_f32(normals, "normals", 3)
    _need_cuda_f32(alpha, "alpha")
    M = int(xyz.shape[0])
    L = lib()
    buf = _alloc_bytes(L.lsgcpd_target_bytes(M), xyz.device)
    ws = _alloc_bytes(L.lsgcpd_pack_workspace_bytes(M), xyz.device)
    info = TargetInfo()
    _check(L.lsgcpd_pack_target(xyz.data_ptr(), normals.data_ptr(), alpha.data_ptr(), M, volume_margin,
                                buf.data_ptr(), ws.data_ptr(), ws.numel(), ctypes.byref(info), _stream_ptr(stream)))
    return _target_from_info(buf, M, info)


class EstepRunner:
    """Reusable lsgcpd_estep launcher (workspace and record allocated once)."""

    def __init__(self, target: Target, src, out=None):
        import torch
        _need_cuda_f32(src, "src", 3)
        self.target, self.src = target, src
        self.N = int(src.shape[0])
        L = lib()
        self.ws = _alloc_bytes(L.lsgcpd_estep_workspace_bytes(target.M, self.N), src.device)
        self.rec = out if out is not None else torch.empty((self.N, REC), dtype=torch.float32, device=src.device)

    def __call__(self, R, t, sigma2: float, w: float, volume: Optional[float] = None, consistent: bool = True,
                 stream=None, eta: Optional[float] = None, src_conf=None, group: str = "se3"):
        Ra, Rp = _darr(R, 9)
        ta, tp = _darr(t, 3)
        V = self.target.volume if volume is None else float(volume)
        if eta is None and src_conf is None and _group(group) == 0:
            _check(lib().lsgcpd_estep(self.target.buf.data_ptr(), self.target.M, self.src.data_ptr(), self.N, Rp, tp,
                                      float(sigma2), float(w), V, int(bool(consistent)), self.rec.data_ptr(),
                                      self.ws.data_ptr(), self.ws.numel(), _stream_ptr(stream)))
        else:
            p = EmParams()
            lib().lsgcpd_em_params_default(ctypes.byref(p))
            p.w = float(w)
            p.consistent_normalizer = int(bool(consistent))
            p.eta = -1.0 if eta is None else float(eta)
            p.d_src_conf = _conf_ptr(src_conf, self.N)
            p.group = _group(group)
            _check(lib().lsgcpd_estep_ex(self.target.buf.data_ptr(), self.target.M, self.src.data_ptr(), self.N, Rp, tp,
                                         float(sigma2), ctypes.byref(p), V, self.rec.data_ptr(), self.ws.data_ptr(),
                                         self.ws.numel(), _stream_ptr(stream)))
        return self.rec


def estep(target: Target, src, R, t, sigma2: float, w: float, volume: Optional[float] = None,
          consistent: bool = True, stream=None, eta: Optional[float] = None, src_conf=None, group: str = "se3"):
    """lsgcpd_estep (or lsgcpd_estep_ex with eta / src_conf / group) → [N,16] float32 CUDA record tensor."""
    return EstepRunner(target, src)(R, t, sigma2, w, volume, consistent, stream, eta, src_conf, group)


def _group(group) -> int:
    """Transformation group of the M step: "se3" (rigid, default) or "affine"."""
    if group in ("se3", 0, None):
        return 0
    if group in ("affine", 1):
        return 1
    raise ValueError(f"unknown group {group!r}")


def _conf_ptr(conf, n):
    if conf is None:
        return None
    _need_cuda_f32(conf, "src_conf")
    if conf.numel() != n:
        raise ValueError(f"src_conf must have {n} entries")
    return conf.data_ptr()


def set_prior(target: Target, phi, stream=None) -> float:
    """lsgcpd_target_set_prior: π(m) = φ(y_m)/Σφ installed in place (Eq. 8).  Returns Σ π √(1+α)."""
    _need_cuda_f32(phi, "phi")
    if phi.numel() != target.M:
        raise ValueError(f"phi must have {target.M} entries")
    ws = _alloc_bytes(lib().lsgcpd_target_prior_workspace_bytes(target.M), phi.device)
    spc = ctypes.c_double()
    _check(lib().lsgcpd_target_set_prior(target.buf.data_ptr(), target.M, phi.data_ptr(), ws.data_ptr(), ws.numel(),
                                         ctypes.byref(spc), _stream_ptr(stream)))
    return spc.value


def select_confident(xyz, phi, threshold: float, stream=None):
    """lsgcpd_select_confident: (points with φ ≥ threshold, their φ), order preserved."""
    import torch
    _need_cuda_f32(xyz, "xyz", 3)
    _need_cuda_f32(phi, "phi")
    n = int(xyz.shape[0])
    out = torch.empty_like(xyz)
    pout = torch.empty_like(phi)
    ws = _alloc_bytes(lib().lsgcpd_select_workspace_bytes(n), xyz.device)
    k = ctypes.c_int64()
    _check(lib().lsgcpd_select_confident(xyz.data_ptr(), phi.data_ptr(), n, float(threshold), out.data_ptr(),
                                         pout.data_ptr(), ctypes.byref(k), ws.data_ptr(), ws.numel(),
                                         _stream_ptr(stream)))
    return out[: k.value].contiguous(), pout[: k.value].contiguous()


def depth_confidence(xyz, c0: float = 0.0, c1: float = 0.002, z_min: float = 0.4, stream=None):
    """lsgcpd_depth_confidence: φ = e(z_min)/e(z), e(z) = c0 + c1 z² of the camera-frame depth."""
    import torch
    _need_cuda_f32(xyz, "xyz", 3)
    phi = torch.empty(int(xyz.shape[0]), dtype=torch.float32, device=xyz.device)
    _check(lib().lsgcpd_depth_confidence(xyz.data_ptr(), int(xyz.shape[0]), float(c0), float(c1), float(z_min),
                                         phi.data_ptr(), _stream_ptr(stream)))
    return phi


class Comm:
    """NCCL communicator wrapper (one process per GPU); the id is broadcast over torch.distributed."""

    def __init__(self, rank: int, world_size: int, group=None):
        from .dist import broadcast_bytes
        blob = b""
        if rank == 0:
            raw = (ctypes.c_char * 128)()
            _check(lib().lsgcpd_comm_unique_id(ctypes.cast(raw, ctypes.c_void_p)))
            blob = bytes(raw.raw)
        blob = broadcast_bytes(blob, 0, group)
        raw = (ctypes.c_char * 128).from_buffer_copy(blob)
        h = ctypes.c_void_p()
        _check(lib().lsgcpd_comm_init(rank, world_size, ctypes.cast(raw, ctypes.c_void_p), ctypes.byref(h)))
        self.handle = h
        self.rank, self.world_size = rank, world_size

    def close(self):
        if self.handle:
            lib().lsgcpd_comm_destroy(self.handle)
            self.handle = None


class Registrar:
    """Reusable lsgcpd_register launcher (workspace allocated once per shape)."""

    def __init__(self, target: Target, src_local, max_iters: int):
        _need_cuda_f32(src_local, "src_local", 3)
        self.target, self.src = target, src_local
        self.N = int(src_local.shape[0])
        self.max_iters = int(max_iters)
        self.ws = _alloc_bytes(lib().lsgcpd_register_workspace_bytes(target.M, self.N, self.max_iters),
                               src_local.device)

    def __call__(self, w: float = 0.1, newton_max: int = 10, consistent: bool = True, sigma2_init: float = 0.0,
                 sigma2_floor_rel: float = 1e-12, tol: float = 0.0, R0=None, t0=None, volume: float = 0.0,
                 comm: Optional[Comm] = None, traces: bool = False, stream=None, check: bool = True,
                 eta: Optional[float] = None, src_conf=None, group: str = "se3"):
        p = EmParams(w, self.max_iters, newton_max, int(bool(consistent)), sigma2_init, sigma2_floor_rel, tol,
                     -1.0 if eta is None else float(eta), _conf_ptr(src_conf, self.N), _group(group))
        R0a, R0p = _darr(np.eye(3) if R0 is None else R0, 9)
        t0a, t0p = _darr(np.zeros(3) if t0 is None else t0, 3)
        Ro = np.zeros(9)
        to = np.zeros(3)
        s2 = ctypes.c_double()
        it = ctypes.c_int()
        nll = np.zeros(max(self.max_iters, 1)) if traces else None
        sg = np.zeros(self.max_iters + 1) if traces else None
        rc = lib().lsgcpd_register(self.target.buf.data_ptr(), self.target.M, float(volume), self.src.data_ptr(),
                                   self.N, ctypes.byref(p), R0p, t0p, Ro.ctypes.data_as(_dp), to.ctypes.data_as(_dp),
                                   ctypes.byref(s2), ctypes.byref(it),
                                   nll.ctypes.data_as(_dp) if traces else None,
                                   sg.ctypes.data_as(_dp) if traces else None,
                                   comm.handle if comm is not None else None, self.ws.data_ptr(), self.ws.numel(),
                                   _stream_ptr(stream))
        out = {"R": Ro.reshape(3, 3), "t": to, "sigma2": s2.value, "iters": it.value, "status": rc}
        if traces:
            out["nll"] = nll[: it.value]
            out["sigma2_trace"] = sg[: it.value + 1]
        if check and rc not in (0, -5):
            _check(rc)
        return out


def register(target: Target, src_local, max_iters: int, **kw):
    """lsgcpd_register → dict(R, t, sigma2, iters, status[, nll, sigma2_trace])."""
    return Registrar(target, src_local, max_iters)(**kw)


class BatchRegistrar:
    """Reusable lsgcpd_register_batch launcher: B independent problems (targets, sources, optional
    confidences, volumes, initial poses) registered together, one batched E step per EM iteration."""

    def __init__(self, targets, sources, max_iters: int, src_confs=None, volumes=None, R0s=None, t0s=None):
        B = len(targets)
        if len(sources) != B or B < 1:
            raise ValueError("need one source per target")
        self.targets, self.sources = list(targets), list(sources)
        self.confs = list(src_confs) if src_confs is not None else [None] * B
        self.max_iters = int(max_iters)
        arr = (Problem * B)()
        for b, (tg, src) in enumerate(zip(self.targets, self.sources)):
            _need_cuda_f32(src, "source", 3)
            pb = arr[b]
            pb.d_target = tg.buf.data_ptr()
            pb.M = tg.M
            pb.d_src = src.data_ptr()
            pb.N = int(src.shape[0])
            pb.d_src_conf = _conf_ptr(self.confs[b], pb.N)
            pb.volume = 0.0 if volumes is None else float(volumes[b])
            R0 = np.eye(3) if R0s is None else np.asarray(R0s[b], dtype=np.float64)
            t0 = np.zeros(3) if t0s is None else np.asarray(t0s[b], dtype=np.float64)
            for i in range(9):
                pb.R0[i] = float(R0.reshape(9)[i])
            for i in range(3):
                pb.t0[i] = float(t0[i])
        self.problems, self.B = arr, B
        nbytes = lib().lsgcpd_register_batch_workspace_bytes(arr, B, self.max_iters)
        if nbytes == 0:
            raise LsgcpdError(-1, "invalid batch")
        self.ws = _alloc_bytes(nbytes, self.sources[0].device)

    def __call__(self, w: float = 0.1, newton_max: int = 10, consistent: bool = True, sigma2_init: float = 0.0,
                 sigma2_floor_rel: float = 1e-12, tol: float = 0.0, eta: Optional[float] = None, stream=None,
                 group: str = "se3"):
        p = EmParams(w, self.max_iters, newton_max, int(bool(consistent)), sigma2_init, sigma2_floor_rel, tol,
                     -1.0 if eta is None else float(eta), None, _group(group))
        B = self.B
        R = np.zeros((B, 9))
        t = np.zeros((B, 3))
        s2 = np.zeros(B)
        it = (ctypes.c_int * B)()
        stt = (ctypes.c_int * B)()
        _check(lib().lsgcpd_register_batch(self.problems, B, ctypes.byref(p), R.ctypes.data_as(_dp),
                                           t.ctypes.data_as(_dp), s2.ctypes.data_as(_dp), it, stt,
                                           self.ws.data_ptr(), self.ws.numel(), _stream_ptr(stream)))
        return {"R": R.reshape(B, 3, 3), "t": t, "sigma2": s2, "iters": np.array(it[:]), "status": np.array(stt[:])}


def register_batch(targets, sources, max_iters: int, src_confs=None, volumes=None, R0s=None, t0s=None, **kw):
    """lsgcpd_register_batch → dict(R [B,3,3], t [B,3], sigma2 [B], iters [B], status [B])."""
    return BatchRegistrar(targets, sources, max_iters, src_confs, volumes, R0s, t0s)(**kw)


def set_option(name: str, value) -> None:
    """lsgcpd_set_option: run-time knobs for diagnostics and tests (tc, estep_variant, halves, no_fuse,
    graph_cache, no_graph, tile_gate; include/lsgcpd.h)."""
    _check(lib().lsgcpd_set_option(name.encode(), float(value)))


def get_option(name: str) -> float:
    v = ctypes.c_double()
    _check(lib().lsgcpd_get_option(name.encode(), ctypes.byref(v)))
    return v.value


class options:
    """Context manager: set options for a block and restore the previous values, e.g.
    ``with lsg.options(tc=0, estep_variant=1): ...``"""

    def __init__(self, **kw):
        self.kw = kw
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *a):
        for k, v in self.old.items():
            set_option(k, v)


def register_shards(target: Target, sources, max_iters: int, w: float = 0.1, newton_max: int = 10,
                    consistent: bool = True, sigma2_init: float = 0.0, sigma2_floor_rel: float = 1e-12,
                    R0=None, t0=None, volume: float = 0.0, stream=None):
    """lsgcpd_register_shards: the multi-GPU protocol (shard moments all-reduced every EM iteration, Newton
    per rank) with len(sources) shards on one device → dict(R [G,3,3], t [G,3], sigma2 [G], iters [G])."""
    G = len(sources)
    for x in sources:
        _need_cuda_f32(x, "source shard", 3)
    Ns = (ctypes.c_int64 * G)(*[int(x.shape[0]) for x in sources])
    ptrs = (ctypes.c_void_p * G)(*[x.data_ptr() for x in sources])
    stride = max(lib().lsgcpd_register_workspace_bytes(target.M, int(n), int(max_iters)) for n in Ns)
    stride = (stride + 255) // 256 * 256
    ws = _alloc_bytes(stride * G, sources[0].device)
    p = EmParams(w, int(max_iters), newton_max, int(bool(consistent)), sigma2_init, sigma2_floor_rel, 0.0, -1.0,
                 None, 0)
    R0a, R0p = _darr(np.eye(3) if R0 is None else R0, 9)
    t0a, t0p = _darr(np.zeros(3) if t0 is None else t0, 3)
    R = np.zeros((G, 9))
    t = np.zeros((G, 3))
    s2 = np.zeros(G)
    it = (ctypes.c_int * G)()
    _check(lib().lsgcpd_register_shards(target.buf.data_ptr(), target.M, float(volume), ptrs, Ns, G, ctypes.byref(p),
                                        R0p, t0p, R.ctypes.data_as(_dp), t.ctypes.data_as(_dp),
                                        s2.ctypes.data_as(_dp), it, ws.data_ptr(), stride, _stream_ptr(stream)))
    return {"R": R.reshape(G, 3, 3), "t": t, "sigma2": s2, "iters": np.array(it[:])}

