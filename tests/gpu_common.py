"""Shared fixtures for -m gpu tests: seeded inputs, the oracle's prepared target rounded to FP32."""
import functools

import numpy as np

import oracle
import synth


@functools.lru_cache(maxsize=8)
def workload(name):
    return synth.make(name)


@functools.lru_cache(maxsize=8)
def oracle_target32(name):
    """The oracle's prepared target with n and α rounded to FP32 (the inputs both sides share)."""
    wl = workload(name)
    tg = oracle.prepare_target(wl.target, wl.knn_k)
    n32 = tg["normals"].astype(np.float32)
    a32 = tg["alpha"].astype(np.float32)
    V, ext = oracle.working_volume(wl.target)
    return wl, n32, a32, V, ext


def to_dev(a, dtype=None):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
