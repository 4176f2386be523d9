"""Affine registration (the Lie-group Newton M step with the aff(3) basis):
the GPU moment-form Newton on GA⁺(3) vs the oracle's per-point form (oracle/affine.py), exact recovery of a
noiseless affine transform, the E step at a non-orthogonal linear part, and the batched path."""
import numpy as np
import pytest

import oracle
import synth
from tests.gpu_common import oracle_target32, to_dev, workload
from tests.parity import assert_record_parity, transformed

pytestmark = pytest.mark.gpu

A_GT = np.array([[1.08, 0.05, 0.0], [-0.03, 0.95, 0.04], [0.02, 0.0, 1.03]])
T_GT = np.array([0.02, -0.03, 0.01])


def _close_affine(A, t, Ar, tr, ext, tol=1e-4):
    dA = np.linalg.norm(np.asarray(A) - np.asarray(Ar))
    dt = np.linalg.norm(np.asarray(t) - np.asarray(tr))
    assert dA <= tol and dt <= tol * ext, (dA, dt)


def test_affine_estep_at_a_non_orthogonal_linear_part():
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    tgt = lsg.pack_target(to_dev(wl.target), to_dev(n32), to_dev(a32))
    A = wl.R_expected @ A_GT
    for s2 in (1e-3, 1e-5):
        rec = lsg.estep(tgt, to_dev(wl.source), A, wl.t_expected, s2, wl.w, V, group="affine").cpu().numpy()
        ora = oracle.estep(wl.target, n32, a32, wl.source, A, wl.t_expected, s2, wl.w, V)
        assert_record_parity(rec, ora, wl.target, a32, what=f"affine E step s2={s2}",
                             Xh=transformed(wl.source, A, wl.t_expected), s2=s2)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.estep(tgt, to_dev(wl.source), A, wl.t_expected, 1e-3, wl.w, V)          # not a rotation
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.estep(tgt, to_dev(wl.source), -np.eye(3), wl.t_expected, 1e-3, wl.w, V, group="affine")


def test_affine_registration_vs_oracle():
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    tgt = lsg.pack_target(to_dev(wl.target), to_dev(n32), to_dev(a32))
    gpu = lsg.register(tgt, to_dev(wl.source), wl.iters, w=wl.w, volume=V, group="affine", traces=True)
    t64 = {"Y": wl.target.astype(np.float64), "normals": n32.astype(np.float64), "alpha": a32.astype(np.float64)}
    ora = oracle.register(t64, wl.source, wl.w, wl.iters, V, ext, group="affine")
    _close_affine(gpu["R"], gpu["t"], ora["R"], ora["t"], ext)
    np.testing.assert_allclose(gpu["sigma2_trace"], ora["trace"]["sigma2"], rtol=1e-3)
    np.testing.assert_allclose(gpu["nll"], ora["trace"]["nll"], rtol=1e-5, atol=1e-3)


def test_affine_exact_recovery_of_a_noiseless_transform():
    import paper_2103_15039_b200 as lsg
    wl = workload("tiny_noiseless")
    Xs = ((wl.target.astype(np.float64) - T_GT) @ np.linalg.inv(A_GT).T).astype(np.float32)
    tgt = lsg.prepare_target(to_dev(wl.target), wl.knn_k)
    out = lsg.register(tgt, to_dev(Xs), 80, w=0.1, group="affine")
    _close_affine(out["R"], out["t"], A_GT, T_GT, tgt.extent, tol=1e-5)


def test_affine_batch_matches_single_problems():
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(3, 500, seed=13)
    tgts = [lsg.prepare_target(to_dev(w.target), w.knn_k) for w in wls]
    out = lsg.register_batch(tgts, [to_dev(w.source) for w in wls], 25, w=0.1, group="affine")
    for b, (w, tg) in enumerate(zip(wls, tgts)):
        single = lsg.register(tg, to_dev(w.source), 25, w=0.1, group="affine")
        _close_affine(out["R"][b], out["t"][b], single["R"], single["t"], tg.extent, tol=1e-5)
