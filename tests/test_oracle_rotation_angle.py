"""Pins for oracle.se3.rotation_angle — the rotation-error metric behind every registration parity bar.

PAPER.md:534 (§4.4): "The rotation error Δθ is the angle of the axis-angle parameterization of the relative
rotation between the ground truth and the registration result."  The checker is pinned here against
things other than itself: rotation matrices built by scipy's `Rotation.from_rotvec` (a library routine,
not the oracle's Rodrigues code), explicit axis rotations cos/sin written out, the special values 0 and π,
and the invariances an angle metric must have.  A plausible slip (trace − 1 without the /2, arccos losing
small angles, a dropped skew term) fails at least one case.
"""
import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from oracle import se3

ANGLES = [1e-9, 1e-4, 0.3, 2.0, np.pi - 1e-6]


def _axes(seed, k):
    a = np.random.default_rng(seed).standard_normal((k, 3))
    return a / np.linalg.norm(a, axis=1, keepdims=True)


@pytest.mark.parametrize("theta", ANGLES)
def test_angle_of_scipy_rotvec(theta):
    for ax in _axes(11, 8):
        R = Rotation.from_rotvec(theta * ax).as_matrix()
        got = se3.rotation_angle(R)
        # relative accuracy at small angles (arctan2 of the skew part), absolute near π
        assert abs(got - theta) <= 1e-9 * theta + 2e-12, (theta, got)


@pytest.mark.parametrize("theta", ANGLES)
def test_angle_of_oracle_exp_matches_rotvec(theta):
    # the oracle's own se3.exp must agree with the library rotation, so R_gpu^T R_ora angles built from it are
    # the P:534 metric
    for ax in _axes(12, 4):
        R, _ = se3.exp(np.concatenate([theta * ax, np.zeros(3)]))
        np.testing.assert_allclose(R, Rotation.from_rotvec(theta * ax).as_matrix(), atol=1e-14)
        assert abs(se3.rotation_angle(R) - theta) <= 1e-9 * theta + 2e-12


def test_explicit_axis_rotations_and_special_values():
    for th in (0.0, 0.25, 1.0, 3.0):
        c, s = np.cos(th), np.sin(th)
        Rx = np.array([[1, 0, 0], [0, c, -s], [0, s, c]])
        Ry = np.array([[c, 0, s], [0, 1, 0], [-s, 0, c]])
        Rz = np.array([[c, -s, 0], [s, c, 0], [0, 0, 1]])
        for R in (Rx, Ry, Rz, Rx.T, Rz.T):
            assert abs(se3.rotation_angle(R) - th) < 1e-14
    assert se3.rotation_angle(np.eye(3)) == 0.0
    for d in ([1, -1, -1], [-1, 1, -1], [-1, -1, 1]):   # half turns: trace = -1
        assert abs(se3.rotation_angle(np.diag(d).astype(float)) - np.pi) < 1e-15


def test_relative_rotation_metric_invariances():
    rng = np.random.default_rng(13)
    for _ in range(20):
        A = Rotation.from_rotvec(rng.standard_normal(3)).as_matrix()
        B = Rotation.from_rotvec(rng.standard_normal(3)).as_matrix()
        Q = Rotation.from_rotvec(rng.standard_normal(3)).as_matrix()
        d = se3.rotation_angle(A.T @ B)
        # symmetric, conjugation-invariant, equals the library's magnitude of the relative rotation
        assert abs(d - se3.rotation_angle(B.T @ A)) < 1e-12
        assert abs(d - se3.rotation_angle(Q @ A.T @ B @ Q.T)) < 1e-12
        assert abs(d - Rotation.from_matrix(A.T @ B).magnitude()) < 1e-10
        assert 0.0 <= d <= np.pi
    # composition about one axis adds angles (below π)
    ax = _axes(14, 1)[0]
    Ra = Rotation.from_rotvec(0.4 * ax).as_matrix()
    Rb = Rotation.from_rotvec(1.1 * ax).as_matrix()
    assert abs(se3.rotation_angle(Ra @ Rb) - 1.5) < 1e-14
