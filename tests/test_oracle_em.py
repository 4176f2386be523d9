"""Pins for the oracle EM loop: monotone NLL (EM property), exact recovery of a noiseless transform,
self-registration → identity, and A→B / B→A consistency."""
import numpy as np
import pytest

import oracle
import synth
from oracle import se3


def test_nll_monotone_tiny():
    wl = synth.make("tiny")
    out = oracle.register_workload(wl, iters=30)
    nll = np.array(out["trace"]["nll"])
    assert np.all(np.diff(nll) <= 1e-9 * np.abs(nll).max()), np.diff(nll).max()
    # noise-limited recovery of the seeded motion: well within 1e-2 rad / 1e-2·extent
    assert se3.rotation_angle(out["R"].T @ wl.R_expected) < 1e-2
    assert np.linalg.norm(out["t"] - wl.t_expected) < 1e-2 * out["extent"]


def test_exact_recovery_noiseless():
    # BJ north star: source = g_gt(target points) → registration returns g_gt⁻¹ exactly (up to σ² floor)
    wl = synth.make("tiny_noiseless")
    out = oracle.register_workload(wl, iters=60)
    assert se3.rotation_angle(out["R"].T @ wl.R_expected) < 1e-7
    assert np.linalg.norm(out["t"] - wl.t_expected) < 1e-7 * out["extent"]


def test_self_registration_is_identity():
    wl = synth.make("tiny")
    tgt = oracle.prepare_target(wl.target, 10)
    V, ext = oracle.working_volume(wl.target)
    out = oracle.register(tgt, wl.target, 0.1, 20, V, ext)
    assert se3.rotation_angle(out["R"]) < 1e-8
    assert np.linalg.norm(out["t"]) < 1e-8 * ext


def test_forward_backward_consistency():
    # g(A→B) ∘ g(B→A) ≈ I (noise-level)
    wl = synth.make("tiny")
    A, B = wl.source, wl.target
    tA, tB = oracle.prepare_target(A, 10), oracle.prepare_target(B, 10)
    VA, eA = oracle.working_volume(A)
    VB, eB = oracle.working_volume(B)
    fwd = oracle.register(tB, A, 0.1, 40, VB, eB)
    bwd = oracle.register(tA, B, 0.1, 40, VA, eA)
    Rc, tc = se3.compose(fwd["R"], fwd["t"], bwd["R"], bwd["t"])
    assert se3.rotation_angle(Rc) < 5e-3
    assert np.linalg.norm(tc) < 5e-3 * eB
