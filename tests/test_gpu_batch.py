"""Batched registrations: lsgcpd_register_batch runs many small problems through one
batched E step per EM iteration.  Each problem's result must meet the north-star registration bar against
the FP64 oracle run on that problem alone (R within 1e-4 rad, t within 1e-4·extent), whatever else is in
the batch; a problem that loses its mass reports ENOMASS without disturbing the others."""
import numpy as np
import pytest

import oracle
import synth
from oracle import se3
from tests.gpu_common import to_dev

pytestmark = pytest.mark.gpu


def _prep(wl):
    import paper_2103_15039_b200 as lsg
    tgt, ann = lsg.prepare_target(to_dev(wl.target), wl.knn_k, annotations=True)
    t64 = {"Y": wl.target.astype(np.float64), "normals": ann["normals"].cpu().numpy().astype(np.float64),
           "alpha": ann["alpha"].cpu().numpy().astype(np.float64)}
    return tgt, t64


def _close(R, t, Rr, tr, ext, tol=1e-4):
    ang = se3.rotation_angle(np.asarray(R).T @ np.asarray(Rr))
    assert ang <= tol and np.linalg.norm(np.asarray(t) - np.asarray(tr)) <= tol * ext, (ang, t, tr)


def test_batch_matches_the_oracle_per_problem():
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(7, 700, ragged=True)
    preps = [_prep(w) for w in wls]
    iters = 30
    out = lsg.register_batch([p[0] for p in preps], [to_dev(w.source) for w in wls], iters, w=0.1)
    assert np.all(out["iters"] == iters) and np.all(out["status"] == 0)
    for b, (w, (tgt, t64)) in enumerate(zip(wls, preps)):
        ora = oracle.register(t64, w.source, 0.1, iters, tgt.volume, tgt.extent)
        _close(out["R"][b], out["t"][b], ora["R"], ora["t"], tgt.extent)
        assert out["sigma2"][b] == pytest.approx(ora["sigma2"], rel=1e-3)
        single = lsg.register(tgt, to_dev(w.source), iters, w=0.1)
        _close(out["R"][b], out["t"][b], single["R"], single["t"], tgt.extent, tol=1e-5)


def test_batch_isolates_a_failing_problem():
    # a problem that loses its inlier mass stops with ENOMASS after 3 iterations, one with a NaN source is
    # refused with EINVAL; every other problem lands
    # where its single-problem lsgcpd_register lands (that one runs the small-problem CUDA-core E step, the
    # batch the tensor-core one: equal up to FP32 summation order)
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(4, 600, seed=11)
    tgts = [_prep(w)[0] for w in wls]
    srcs = [w.source for w in wls]
    srcs[2] = (srcs[2] + 1e4).astype(np.float32)                     # far away: no inlier mass
    srcs[1] = srcs[1].copy()
    srcs[1][17, 0] = np.nan                                          # refused: EINVAL, never iterated
    out = lsg.register_batch(tgts, [to_dev(s) for s in srcs], 20, w=0.1, sigma2_init=1e-3)
    assert out["status"][2] == -5 and out["iters"][2] == 3
    assert out["status"][1] == -1 and out["iters"][1] == 0
    for b in (0, 3):
        single = lsg.register(tgts[b], to_dev(srcs[b]), 20, w=0.1, sigma2_init=1e-3)
        assert out["status"][b] == 0 and out["iters"][b] == 20
        _close(out["R"][b], out["t"][b], single["R"], single["t"], tgts[b].extent, tol=1e-5)
        assert out["sigma2"][b] == pytest.approx(single["sigma2"], rel=1e-5)


def test_batch_with_eta_and_confidence_vs_oracle():
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(4, 1000, seed=11)
    preps = [_prep(w) for w in wls]
    rng = np.random.default_rng(4)
    confs = [rng.uniform(0.3, 1.0, w.N).astype(np.float32) for w in wls]
    out = lsg.register_batch([p[0] for p in preps], [to_dev(w.source) for w in wls], 30,
                             src_confs=[to_dev(c) for c in confs], eta=0.1)
    for b, w in enumerate(wls):
        tgt, t64 = preps[b]
        ora = oracle.register(t64, w.source, 0.0, 30, tgt.volume, tgt.extent, eta=0.1,
                              phi_x=confs[b].astype(np.float64))
        assert out["status"][b] == 0 and out["iters"][b] == 30
        _close(out["R"][b], out["t"][b], ora["R"], ora["t"], tgt.extent)


def test_batch_invalid_arguments():
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(2, 300, seed=12)
    tgts = [_prep(w)[0] for w in wls]
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.register_batch(tgts, [to_dev(w.source) for w in wls], 5, w=1.0)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.register_batch(tgts, [to_dev(w.source) for w in wls], 5, R0s=[2 * np.eye(3)] * 2)


def test_batch_running_max_mode_and_priors_match_single_registrations():
    # w = 0 puts every problem in the running-max mode (the CUDA-core batched kernel serves them); a target
    # with priors π(m) (Eq. 8) is served by the tensor-core batched kernel: each problem lands where its
    # single-problem lsgcpd_register lands, and priors with the literal normaliser are refused
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(3, 800, seed=17)
    tgts = [_prep(w)[0] for w in wls]
    srcs = [to_dev(w.source) for w in wls]
    out = lsg.register_batch(tgts, srcs, 20, w=0.0)
    for b in range(3):
        single = lsg.register(tgts[b], srcs[b], 20, w=0.0)
        assert out["status"][b] == 0 and single["status"] == 0
        _close(out["R"][b], out["t"][b], single["R"], single["t"], tgts[b].extent, tol=1e-5)
    phi = to_dev(np.random.default_rng(3).uniform(0.2, 1.0, tgts[1].M).astype(np.float32))
    lsg.set_prior(tgts[1], phi)
    out = lsg.register_batch(tgts, srcs, 20, w=0.1)
    single = lsg.register(tgts[1], srcs[1], 20, w=0.1)
    _close(out["R"][1], out["t"][1], single["R"], single["t"], tgts[1].extent, tol=1e-5)
    with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
        lsg.register_batch(tgts, srcs, 5, w=0.1, consistent=False)


def test_batch_literal_normaliser_matches_single_registrations():
    # the batched tensor-core E step's kLiteral instantiation (Eq. 9-10 normaliser, no priors): every problem
    # lands where its single-problem registration with the literal normaliser lands
    import paper_2103_15039_b200 as lsg
    wls = synth.make_batch(3, 900, seed=23)
    tgts = [_prep(w)[0] for w in wls]
    srcs = [to_dev(w.source) for w in wls]
    out = lsg.register_batch(tgts, srcs, 20, w=0.1, consistent=False)
    for b in range(3):
        single = lsg.register(tgts[b], srcs[b], 20, w=0.1, consistent=False)
        assert out["status"][b] == 0 and single["status"] == 0
        _close(out["R"][b], out["t"][b], single["R"], single["t"], tgts[b].extent, tol=1e-5)
