"""GPU parity for the §3.2-3.3 model extensions:
outlier weight from the outlier ratio η (Eq. 7) and confidence filtering (Eq. 8):
component priors π(m) installed in the prepared target (lsgcpd_target_set_prior), per-point outlier
weights w_n from source confidences (lsgcpd_estep_ex / lsgcpd_register), truncation
(lsgcpd_select_confident) and the depth error model (lsgcpd_depth_confidence) — all against the FP64
oracle (oracle/outlier.py, oracle.estep_cf)."""
import numpy as np
import pytest

import oracle
from oracle import outlier as ol, se3
from tests.gpu_common import oracle_target32, to_dev, workload
from tests.parity import assert_record_parity, transformed

pytestmark = pytest.mark.gpu


def _target_with_prior(wl, n32, a32, phi_y):
    import paper_2103_15039_b200 as lsg
    tgt = lsg.pack_target(to_dev(wl.target), to_dev(n32), to_dev(a32))
    spc = lsg.set_prior(tgt, to_dev(phi_y.astype(np.float32)))
    return tgt, spc


@pytest.mark.parametrize("consistent", [True, False])
@pytest.mark.parametrize("mode", ["w0", "w0=0", "eta"])
def test_estep_ex_prior_and_point_weights(consistent, mode):
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("object")
    rng = np.random.default_rng(21)
    phi_y = rng.uniform(0.05, 1.0, wl.M).astype(np.float32)
    phi_y[rng.choice(wl.M, 50, replace=False)] = 0.0                  # removed components
    phi_x = rng.uniform(0.0, 1.0, wl.N).astype(np.float32)
    phi_x[:20] = 0.0                                                   # all-outlier points
    phi_x[20:40] = 1.0
    tgt, spc = _target_with_prior(wl, n32, a32, phi_y)
    if not consistent:   # the Eq. 9-10 literal form has π(m) = 1/M: non-uniform priors are refused
        with pytest.raises(lsg.LsgcpdError, match="EINVAL"):
            lsg.estep(tgt, to_dev(wl.source), np.eye(3), np.zeros(3), 1e-3, 0.1, V, False)
        phi_y = np.ones(wl.M, np.float32)
        spc = lsg.set_prior(tgt, to_dev(phi_y))
    pi = ol.confidence_prior(phi_y.astype(np.float64))
    assert spc == pytest.approx(float(np.dot(pi, np.sqrt(1.0 + a32.astype(np.float64)))), rel=1e-6)
    X = to_dev(wl.source)
    for s2 in (1e-2, 1e-4):
        if mode == "eta":
            w0 = ol.outlier_weight_max(0.15, V, pi, a32, s2, consistent)
            rec = lsg.estep(tgt, X, wl.R_expected, wl.t_expected, s2, 0.0, V, consistent, eta=0.15,
                            src_conf=to_dev(phi_x)).cpu().numpy()
        else:
            w0 = 0.0 if mode == "w0=0" else 0.1
            rec = lsg.estep(tgt, X, wl.R_expected, wl.t_expected, s2, w0, V, consistent,
                            src_conf=to_dev(phi_x)).cpu().numpy()
        wn = ol.point_outlier_weights(w0, phi_x.astype(np.float64))
        ora = oracle.estep_cf(wl.target, n32, a32, pi, wl.source, wn, wl.R_expected, wl.t_expected, s2, V, consistent)
        assert_record_parity(rec, ora, wl.target, a32, what=f"{mode} consistent={consistent} s2={s2}",
                             Xh=transformed(wl.source, wl.R_expected, wl.t_expected), s2=s2)
        assert np.all(rec[:20, 15] == 1.0) and np.all(rec[:20, :14] == 0.0)
        np.testing.assert_allclose(rec[:, 0] + rec[:, 15], 1.0, atol=3e-6)


def test_uniform_prior_restores_the_uniform_model():
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    rng = np.random.default_rng(2)
    tgt, _ = _target_with_prior(wl, n32, a32, rng.uniform(0.1, 1, wl.M))
    lsg.set_prior(tgt, to_dev(np.ones(wl.M, np.float32)))              # idempotent: back to π = 1/M
    for s2 in (1e-3, 1e-5):
        rec = lsg.estep(tgt, to_dev(wl.source), wl.R_expected, wl.t_expected, s2, wl.w, V).cpu().numpy()
        ora = oracle.estep(wl.target, n32, a32, wl.source, wl.R_expected, wl.t_expected, s2, wl.w, V)
        assert_record_parity(rec, ora, wl.target, a32, what=f"uniform again s2={s2}",
                             Xh=transformed(wl.source, wl.R_expected, wl.t_expected), s2=s2)


def test_register_with_eta_and_confidence_vs_oracle():
    import paper_2103_15039_b200 as lsg
    wl, n32, a32, V, ext = oracle_target32("tiny")
    rng = np.random.default_rng(8)
    phi_y = rng.uniform(0.2, 1.0, wl.M)
    phi_x = rng.uniform(0.2, 1.0, wl.N).astype(np.float32)
    tgt, _ = _target_with_prior(wl, n32, a32, phi_y)
    pi = ol.confidence_prior(phi_y.astype(np.float32).astype(np.float64))
    target64 = {"Y": wl.target.astype(np.float64), "normals": n32.astype(np.float64), "alpha": a32.astype(np.float64)}
    for eta in (None, 0.1):
        gpu = lsg.register(tgt, to_dev(wl.source), wl.iters, w=wl.w, volume=V, eta=eta, src_conf=to_dev(phi_x),
                           traces=True)
        ora = oracle.register(target64, wl.source, wl.w, wl.iters, V, ext, eta=eta, prior=pi,
                              phi_x=phi_x.astype(np.float64))
        ang = se3.rotation_angle(gpu["R"].T @ ora["R"])
        assert ang <= 1e-4 and np.linalg.norm(gpu["t"] - ora["t"]) <= 1e-4 * ext, (eta, ang)
        np.testing.assert_allclose(gpu["sigma2_trace"], ora["trace"]["sigma2"], rtol=1e-3)
        np.testing.assert_allclose(gpu["nll"], ora["trace"]["nll"], rtol=1e-5, atol=1e-3)


def test_depth_confidence_and_truncation_match_the_oracle():
    import paper_2103_15039_b200 as lsg
    wl = workload("rgbd")
    X = to_dev(wl.source)
    phi = lsg.depth_confidence(X).cpu().numpy()
    ref = ol.depth_confidence(wl.source[:, 2].astype(np.float64)).astype(np.float32)
    np.testing.assert_allclose(phi, ref, rtol=2e-7, atol=0)
    thr = np.float32(0.04)
    kept, kphi = lsg.select_confident(X, to_dev(ref), float(thr))
    o_pts, o_phi, keep = ol.truncate(wl.source, ref, thr)          # the decision in FP32 on both sides
    assert kept.shape[0] == int(keep.sum()) and 0 < keep.sum() < wl.N
    np.testing.assert_array_equal(kept.cpu().numpy(), o_pts)
    np.testing.assert_array_equal(kphi.cpu().numpy(), o_phi)


def test_rgbd_confidence_filtered_registration_teacher_forced():
    # the RGBD config with CF: depth confidences, truncation at φ < 0.04 (depth > 2 m), priors on
    # the target, w_n on the source; each EM step of the GPU trajectory checked against the oracle at full size
    import paper_2103_15039_b200 as lsg
    wl = workload("rgbd")
    thr = np.float32(0.04)
    phi_y = ol.depth_confidence(wl.target[:, 2].astype(np.float64)).astype(np.float32)
    phi_x = ol.depth_confidence(wl.source[:, 2].astype(np.float64)).astype(np.float32)
    Y, py, _ = ol.truncate(wl.target, phi_y, thr)
    Xs, px, _ = ol.truncate(wl.source, phi_x, thr)
    tgt, ann = lsg.prepare_target(to_dev(Y), wl.knn_k, annotations=True)
    lsg.set_prior(tgt, to_dev(py))
    n64 = ann["normals"].cpu().numpy().astype(np.float64)
    a64 = ann["alpha"].cpu().numpy().astype(np.float64)
    pi = ol.confidence_prior(py.astype(np.float64))
    X = to_dev(Xs)
    C = to_dev(px)
    idx = np.sort(np.random.default_rng(3).choice(Xs.shape[0], 1024, replace=False))
    floor = 1e-12 * tgt.extent ** 2
    for k in (1, 10, 30):
        st = lsg.Registrar(tgt, X, k)(w=wl.w, src_conf=C)
        nxt = lsg.Registrar(tgt, X, k + 1)(w=wl.w, src_conf=C)
        R, t, s2 = st["R"], st["t"], st["sigma2"]
        rec = lsg.estep(tgt, X, R, t, s2, wl.w, tgt.volume, src_conf=C).cpu().numpy()
        wn = ol.point_outlier_weights(wl.w, px[idx].astype(np.float64))
        ora = oracle.estep_cf(Y, n64, a64, pi, Xs[idx], wn, R, t, s2, tgt.volume)
        assert_record_parity(rec[idx], ora, Y, a64, what=f"rgbd-CF E step at state {k}",
                             Xh=transformed(Xs[idx], R, t), s2=s2)
        R1, t1, s21, _ = oracle.mstep(Xs, rec, R, t, s2, tgt.extent, 10, floor)
        assert se3.rotation_angle(np.asarray(nxt["R"]).T @ R1) <= 1e-4
        assert np.linalg.norm(np.asarray(nxt["t"]) - t1) <= 1e-4 * tgt.extent
        assert abs(nxt["sigma2"] - s21) <= 1e-6 * s21


def test_rgbd_confidence_filtered_registration_vs_golden():
    # the whole RGBD-CF pipeline (NEXT-2) against the FP64 oracle's (oracle/make_golden.py rgbd_cf): the
    # truncated clouds, the GPU-prepared target with priors π(m), per-point w_n, 50 EM iterations
    import json
    import os
    import paper_2103_15039_b200 as lsg
    from oracle.make_golden import digest
    path = os.path.join(os.path.dirname(__file__), "golden", "rgbd_cf_oracle.json")
    g = json.load(open(path))
    wl = workload("rgbd")
    thr = np.float32(0.04)
    Y, py, _ = ol.truncate(wl.target, ol.depth_confidence(wl.target[:, 2].astype(np.float64)).astype(np.float32), thr)
    X, px, _ = ol.truncate(wl.source, ol.depth_confidence(wl.source[:, 2].astype(np.float64)).astype(np.float32), thr)
    assert (digest(Y), digest(X)) == (g["target_sha"], g["source_sha"]), "inputs changed"
    tgt = lsg.prepare_target(to_dev(Y), wl.knn_k)
    assert tgt.volume == pytest.approx(g["V"], rel=1e-6)
    lsg.set_prior(tgt, to_dev(py))
    out = lsg.register(tgt, to_dev(X), g["iters"], w=wl.w, src_conf=to_dev(px))
    assert out["status"] == 0 and out["iters"] == g["iters"]
    ang = se3.rotation_angle(np.asarray(out["R"]).T @ np.array(g["R"]))
    assert ang <= 1e-4, ang
    assert np.linalg.norm(np.asarray(out["t"]) - np.array(g["t"])) <= 1e-4 * g["extent"]
    assert out["sigma2"] == pytest.approx(g["sigma2"], rel=1e-3)
