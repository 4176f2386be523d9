"""ctypes loader for the FP64 C oracle (oracle/lsgcpd_oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
import anything under oracle/.  The product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lsgcpd_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp, IEEE semantics: no -ffast-math)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_SO)
            dp = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            L.ora_estep.argtypes = [dp, dp, dp, i64, dp, i64, dp, dp, ctypes.c_double, ctypes.c_double,
                                    ctypes.c_double, ctypes.c_int, dp, ctypes.c_int]
            L.ora_estep.restype = None
            L.ora_estep_cf.argtypes = [dp, dp, dp, dp, i64, dp, dp, i64, dp, dp, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_int, dp, ctypes.c_int]
            L.ora_estep_cf.restype = None
            L.ora_posterior.argtypes = [dp, dp, dp, i64, dp, i64, dp, dp, ctypes.c_double, ctypes.c_double,
                                        ctypes.c_double, ctypes.c_int, dp, dp]
            L.ora_posterior.restype = None
            L.ora_knn.argtypes = [dp, i64, ctypes.c_void_p, i64, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                  ctypes.c_int]
            L.ora_knn.restype = None
            L.ora_sum_sq_pairs.argtypes = [dp, i64, dp, i64, ctypes.c_int]
            L.ora_sum_sq_pairs.restype = ctypes.c_double
            L.ora_max_threads.argtypes = []
            L.ora_max_threads.restype = ctypes.c_int
            _lib = L
    return _lib


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
