"""Seeded synthetic point-cloud workloads (the five BASELINE.json configs).

This module is shared by the oracle side (tests, golden scripts) and the product
side (bench.py).  It holds NO arithmetic of the LSG-CPD method: it only samples
surfaces, casts sensor rays and applies the ground-truth rigid motion.  Every
parameter the paper or BASELINE.json leaves open is marked "(choice)" and is
recorded in the returned metadata.

The paper's public datasets (Stanford scans P:359-360/P:456, Stanford Lounge
P:481, KITTI 07 P:528) are not used; these seeded shapes stand in for them.

Conventions
-----------
* ``target`` Y (M×3) and ``source`` X (N×3) are float32, C-contiguous.
* ``g_expected`` = (R, t) in float64 is the rigid map that registration should
  return: the one taking source coordinates into the target frame.  For the
  object-style configs the source is g_gt(resample) and g_expected = g_gt⁻¹.
* RNG: numpy PCG64 with ``SeedSequence(seed).spawn(k)`` sub-streams.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, Optional

import numpy as np

CONFIG_NAMES = ("tiny", "object", "rgbd", "lidar", "scale")
SEEDS = {"tiny": 1, "object": 2, "rgbd": 3, "lidar": 4, "scale": 5}


@dataclasses.dataclass
class Workload:
    name: str
    target: np.ndarray            # (M,3) float32
    source: np.ndarray            # (N,3) float32
    R_expected: np.ndarray        # (3,3) float64
    t_expected: np.ndarray        # (3,)  float64
    w: float
    iters: int
    knn_k: int
    target_inlier: np.ndarray     # (M,) bool
    source_inlier: np.ndarray     # (N,) bool
    meta: Dict

    @property
    def M(self) -> int:
        return int(self.target.shape[0])

    @property
    def N(self) -> int:
        return int(self.source.shape[0])


# ----------------------------------------------------------------------------
# small geometric helpers (sampling / rigid motion only)
# ----------------------------------------------------------------------------

def _unit(rng: np.random.Generator, n: Optional[int] = None) -> np.ndarray:
    """Uniform direction(s) on S² (normalised standard Gaussian)."""
    v = rng.standard_normal((3,) if n is None else (n, 3))
    return v / np.linalg.norm(v, axis=-1, keepdims=True)


def axis_angle(axis: np.ndarray, angle: float) -> np.ndarray:
    """Rotation matrix for a unit axis and angle (Rodrigues), float64."""
    a = np.asarray(axis, dtype=np.float64)
    a = a / np.linalg.norm(a)
    K = np.array([[0.0, -a[2], a[1]], [a[2], 0.0, -a[0]], [-a[1], a[0], 0.0]])
    return np.eye(3) + np.sin(angle) * K + (1.0 - np.cos(angle)) * (K @ K)


def _rot_z(angle: float) -> np.ndarray:
    c, s = np.cos(angle), np.sin(angle)
    return np.array([[c, -s, 0.0], [s, c, 0.0], [0.0, 0.0, 1.0]])


def _apply(R: np.ndarray, t: np.ndarray, P: np.ndarray) -> np.ndarray:
    return P @ R.T + t


def _inverse(R: np.ndarray, t: np.ndarray):
    return R.T.copy(), -(R.T @ t)


def _f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# ----------------------------------------------------------------------------
# surface samplers
# ----------------------------------------------------------------------------

def sample_cube_surface(rng: np.random.Generator, n: int, half: float = 0.5) -> np.ndarray:
    """Uniform on the surface of [-half, half]^3: face uniform among 6, (u,v) uniform."""
    face = rng.integers(0, 6, size=n)
    uv = rng.uniform(-half, half, size=(n, 2))
    P = np.empty((n, 3))
    axis = face // 2
    sign = np.where(face % 2 == 0, -half, half)
    for a in range(3):
        m = axis == a
        others = [b for b in range(3) if b != a]
        P[m, a] = sign[m]
        P[m, others[0]] = uv[m, 0]
        P[m, others[1]] = uv[m, 1]
    return P


def sample_torus(rng: np.random.Generator, n: int, R: float, r: float, center) -> np.ndarray:
    """Area-uniform torus (axis z) by rejection on the area element (R + r cos v)."""
    out = []
    need = n
    while need > 0:
        m = int(need * 2.2) + 16
        u = rng.uniform(0, 2 * np.pi, m)
        v = rng.uniform(0, 2 * np.pi, m)
        acc = rng.uniform(0, 1, m) < (R + r * np.cos(v)) / (R + r)
        u, v = u[acc], v[acc]
        pts = np.stack([(R + r * np.cos(v)) * np.cos(u), (R + r * np.cos(v)) * np.sin(u), r * np.sin(v)], axis=1)
        out.append(pts[:need])
        need -= len(out[-1])
    return np.concatenate(out, axis=0) + np.asarray(center, dtype=np.float64)


def sample_object_scene(rng: np.random.Generator, n: int) -> np.ndarray:
    """Torus (R=1, r=0.3, centre (0,0,0.3) (choice)) ∪ plane z=0 on [-1,1]² (choice), area-proportional."""
    Rt, rt = 1.0, 0.3
    a_torus = 4 * np.pi ** 2 * Rt * rt
    a_plane = 4.0
    n_torus = rng.binomial(n, a_torus / (a_torus + a_plane))
    torus = sample_torus(rng, n_torus, Rt, rt, (0.0, 0.0, 0.3))
    plane = np.column_stack([rng.uniform(-1, 1, n - n_torus), rng.uniform(-1, 1, n - n_torus), np.zeros(n - n_torus)])
    P = np.concatenate([torus, plane], axis=0)
    return P[rng.permutation(n)]


def sample_patches_spheres(rng_layout: np.random.Generator, rng_pts: np.random.Generator, n: int,
                           n_patch: int = 64, n_sphere: int = 64) -> np.ndarray:
    """Mixture of square planar patches and spheres in the unit cube, area-proportional."""
    pc = rng_layout.uniform(-0.4, 0.4, (n_patch, 3))
    pn = _unit(rng_layout, n_patch)
    side = rng_layout.uniform(0.05, 0.25, n_patch)                 # (choice)
    sc = rng_layout.uniform(-0.4, 0.4, (n_sphere, 3))
    rad = rng_layout.uniform(0.02, 0.08, n_sphere)                 # (choice)
    # orthonormal in-plane basis per patch
    helper = np.where(np.abs(pn[:, :1]) < 0.9, np.array([[1.0, 0, 0]]), np.array([[0, 1.0, 0]]))
    e1 = np.cross(pn, helper)
    e1 /= np.linalg.norm(e1, axis=1, keepdims=True)
    e2 = np.cross(pn, e1)
    areas = np.concatenate([side ** 2, 4 * np.pi * rad ** 2])
    comp = rng_pts.choice(len(areas), size=n, p=areas / areas.sum())
    P = np.empty((n, 3))
    isp = comp < n_patch
    k = comp[isp]
    uv = rng_pts.uniform(-0.5, 0.5, (isp.sum(), 2)) * side[k, None]
    P[isp] = pc[k] + uv[:, :1] * e1[k] + uv[:, 1:] * e2[k]
    ks = comp[~isp] - n_patch
    P[~isp] = sc[ks] + rad[ks, None] * _unit(rng_pts, int((~isp).sum()))
    return P


# ----------------------------------------------------------------------------
# ray casting (RGBD room, LiDAR street)
# ----------------------------------------------------------------------------

def _ray_planes_boxes(origin, dirs, planes, boxes):
    """Nearest positive hit along rays.  planes: list of (axis, value, bounds[(lo,hi)x3]);
    boxes: (B,2,3) AABBs.  Returns t (inf where miss)."""
    n = dirs.shape[0]
    best = np.full(n, np.inf)
    with np.errstate(divide="ignore", invalid="ignore"):
        for axis, value, bounds in planes:
            d = dirs[:, axis]
            t = (value - origin[axis]) / d
            hit = origin + t[:, None] * dirs
            ok = (t > 1e-9) & np.isfinite(t)
            for a in range(3):
                if a == axis:
                    continue
                lo, hi = bounds[a]
                ok &= (hit[:, a] >= lo) & (hit[:, a] <= hi)
            best = np.where(ok & (t < best), t, best)
        for b in boxes:
            t1 = (b[0] - origin) / dirs
            t2 = (b[1] - origin) / dirs
            tmin = np.nanmax(np.minimum(t1, t2), axis=1)
            tmax = np.nanmin(np.maximum(t1, t2), axis=1)
            ok = (tmax >= tmin) & (tmin > 1e-9)
            best = np.where(ok & (tmin < best), tmin, best)
    return best


def _ray_cylinders(origin, dirs, cyl_xy, radius, height):
    """Nearest hit with vertical cylinders (side surface, z in [0, height])."""
    n = dirs.shape[0]
    best = np.full(n, np.inf)
    dx, dy = dirs[:, 0], dirs[:, 1]
    a = dx * dx + dy * dy
    with np.errstate(divide="ignore", invalid="ignore"):
        for cx, cy in cyl_xy:
            ox, oy = origin[0] - cx, origin[1] - cy
            b = 2 * (ox * dx + oy * dy)
            c = ox * ox + oy * oy - radius * radius
            disc = b * b - 4 * a * c
            ok = disc >= 0
            sq = np.sqrt(np.where(ok, disc, 0.0))
            t = (-b - sq) / (2 * a)
            z = origin[2] + t * dirs[:, 2]
            ok &= (t > 1e-9) & (z >= 0) & (z <= height)
            best = np.where(ok & (t < best), t, best)
    return best


def _camera_basis(pitch_deg: float) -> np.ndarray:
    """Camera→world rotation for a camera looking +y (world z up), pitched down by pitch_deg.
    Camera frame: x right, y down, z forward."""
    p = np.deg2rad(pitch_deg)
    fwd = np.array([0.0, np.cos(p), -np.sin(p)])
    right = np.array([1.0, 0.0, 0.0])
    down = np.cross(fwd, right)
    return np.column_stack([right, down, fwd])


def _rgbd_scan(rng_noise, R_wc, c_w, planes, boxes, W=320, H=240, f=285.0, cx=159.5, cy=119.5,
               zmin=0.4, zmax=8.0):
    u, v = np.meshgrid(np.arange(W, dtype=np.float64), np.arange(H, dtype=np.float64))
    d_c = np.stack([(u.ravel() - cx) / f, (v.ravel() - cy) / f, np.ones(W * H)], axis=1)
    d_w = d_c @ R_wc.T
    t = _ray_planes_boxes(c_w, d_w, planes, boxes)
    z = t  # d_c.z == 1 so the ray parameter is the depth
    valid = np.isfinite(z) & (z >= zmin) & (z <= zmax)
    z = z[valid]
    z_noisy = z + rng_noise.standard_normal(z.shape) * 0.002 * z ** 2
    return d_c[valid] * z_noisy[:, None]


def _lidar_scan(rng_noise, R_ws, c_w, cyl_xy, rings=64, az=1800, el_hi=2.0, el_lo=-24.8, max_range=120.0):
    el = np.deg2rad(np.linspace(el_hi, el_lo, rings))
    a = np.deg2rad(np.arange(az) * (360.0 / az))
    E, A = np.meshgrid(el, a, indexing="ij")
    d_s = np.stack([np.cos(E) * np.cos(A), np.cos(E) * np.sin(A), np.sin(E)], axis=-1).reshape(-1, 3)
    d_w = d_s @ R_ws.T
    big = 1e4
    planes = [
        (2, 0.0, [(-big, big), (-big, big), (0, 0)]),         # ground
        (1, 8.0, [(-big, big), (0, 0), (0.0, 12.0)]),          # facade y=+8, height 12 m (choice)
        (1, -8.0, [(-big, big), (0, 0), (0.0, 12.0)]),         # facade y=-8
    ]
    t = _ray_planes_boxes(c_w, d_w, planes, np.zeros((0, 2, 3)))
    tc = _ray_cylinders(c_w, d_w, cyl_xy, 0.15, 4.0)            # height 4 m (choice)
    t = np.minimum(t, tc)
    valid = np.isfinite(t) & (t <= max_range)
    r = t[valid] + rng_noise.standard_normal(int(valid.sum())) * 0.02
    return d_s[valid] * r[:, None]


def _add_uniform_outliers(rng, P, frac, lo=None, hi=None):
    n_out = int(round(frac * P.shape[0]))
    if lo is None:
        lo, hi = P.min(axis=0), P.max(axis=0)
    O = rng.uniform(lo, hi, (n_out, 3))
    allp = np.concatenate([P, O], axis=0)
    inl = np.concatenate([np.ones(P.shape[0], bool), np.zeros(n_out, bool)])
    perm = rng.permutation(allp.shape[0])
    return allp[perm], inl[perm]


# ----------------------------------------------------------------------------
# the five configs
# ----------------------------------------------------------------------------

def make_tiny(noiseless: bool = False) -> Workload:
    ss = np.random.SeedSequence(SEEDS["tiny"]).spawn(6)
    r_tgt, r_src, r_noise, r_axis, r_dir, _ = [np.random.Generator(np.random.PCG64(s)) for s in ss]
    Y = sample_cube_surface(r_tgt, 1000)
    if noiseless:
        Xs = Y.copy()
    else:
        Y = Y + r_noise.standard_normal(Y.shape) * 0.005
        Xs = sample_cube_surface(r_src, 1000) + r_noise.standard_normal((1000, 3)) * 0.005
    R_gt = axis_angle(_unit(r_axis), np.deg2rad(30.0))
    t_gt = 0.1 * _unit(r_dir)
    X = _apply(R_gt, t_gt, Xs)
    R_e, t_e = _inverse(R_gt, t_gt)
    n = Y.shape[0]
    return Workload("tiny" + ("_noiseless" if noiseless else ""), _f32(Y), _f32(X), R_e, t_e, 0.1, 50, 10,
                    np.ones(n, bool), np.ones(X.shape[0], bool),
                    {"seed": SEEDS["tiny"], "rot_deg": 30.0, "t_norm": 0.1, "noise_sd": 0.0 if noiseless else 0.005})


def make_object(noiseless: bool = False) -> Workload:
    ss = np.random.SeedSequence(SEEDS["object"]).spawn(8)
    r_tgt, r_src, r_noise, r_axis, r_dir, r_drop_t, r_drop_s, _ = [np.random.Generator(np.random.PCG64(s)) for s in ss]
    n0 = 10000
    Y = sample_object_scene(r_tgt, n0)
    if noiseless:
        Y = Y[np.sort(r_drop_t.permutation(n0)[: n0 - n0 // 20])]
        Xs = Y.copy()
    else:
        Y = Y + r_noise.standard_normal(Y.shape) * 0.003
        Xs = sample_object_scene(r_src, n0) + r_noise.standard_normal((n0, 3)) * 0.003
        Y = Y[np.sort(r_drop_t.permutation(n0)[: n0 - n0 // 20])]
        Xs = Xs[np.sort(r_drop_s.permutation(n0)[: n0 - n0 // 20])]
    R_gt = axis_angle(_unit(r_axis), np.deg2rad(45.0))
    t_gt = 0.2 * _unit(r_dir)
    X = _apply(R_gt, t_gt, Xs)
    R_e, t_e = _inverse(R_gt, t_gt)
    return Workload("object" + ("_noiseless" if noiseless else ""), _f32(Y), _f32(X), R_e, t_e, 0.1, 100, 10,
                    np.ones(Y.shape[0], bool), np.ones(X.shape[0], bool),
                    {"seed": SEEDS["object"], "rot_deg": 45.0, "t_norm": 0.2, "noise_sd": 0.0 if noiseless else 0.003,
                     "torus": {"R": 1.0, "r": 0.3, "center": [0, 0, 0.3]}, "plane": "[-1,1]^2 at z=0", "drop": 0.05})


def make_rgbd() -> Workload:
    ss = np.random.SeedSequence(SEEDS["rgbd"]).spawn(8)
    r_layout, r_noise1, r_noise2, r_dir, r_out1, r_out2, _, _ = [np.random.Generator(np.random.PCG64(s)) for s in ss]
    big = 1e4
    Hh = 2.5
    planes = [
        (2, 0.0, [(-2.5, 2.5), (0.0, 5.0), (0, 0)]),          # floor
        (1, 5.0, [(-2.5, 2.5), (0, 0), (0.0, Hh)]),           # back wall
        (0, -2.5, [(0, 0), (0.0, 5.0), (0.0, Hh)]),           # side walls
        (0, 2.5, [(0, 0), (0.0, 5.0), (0.0, Hh)]),
    ]
    boxes = []
    for _ in range(4):                                         # 4 boxes on the floor (placement is a choice)
        s = r_layout.uniform(0.3, 1.0, 3)
        cx = r_layout.uniform(-2.0, 2.0)
        cy = r_layout.uniform(1.5, 4.5)
        lo = np.array([cx - s[0] / 2, cy - s[1] / 2, 0.0])
        boxes.append(np.stack([lo, lo + s]))
    boxes = np.array(boxes)
    R1 = _camera_basis(5.0)
    c1 = np.array([0.0, 0.3, 1.4])
    R2 = _rot_z(np.deg2rad(10.0)) @ R1
    phi = r_dir.uniform(0, 2 * np.pi)
    c2 = c1 + 0.15 * np.array([np.cos(phi), np.sin(phi), 0.0])
    P1 = _rgbd_scan(r_noise1, R1, c1, planes, boxes)
    P2 = _rgbd_scan(r_noise2, R2, c2, planes, boxes)
    n_valid = (P1.shape[0], P2.shape[0])
    Y, inl_y = _add_uniform_outliers(r_out1, P1, 0.10)
    X, inl_x = _add_uniform_outliers(r_out2, P2, 0.10)
    # expected: map camera-2 coordinates into camera-1 coordinates
    R_e = R1.T @ R2
    t_e = R1.T @ (c2 - c1)
    return Workload("rgbd", _f32(Y), _f32(X), R_e, t_e, 0.1, 50, 10, inl_y, inl_x,
                    {"seed": SEEDS["rgbd"], "valid": n_valid, "f": 285.0, "c": [159.5, 119.5],
                     "cam1": c1.tolist(), "pitch_deg": 5.0, "yaw_deg": 10.0, "shift": 0.15,
                     "boxes": boxes.tolist(), "outlier_frac": 0.10, "z_range": [0.4, 8.0]})


def make_lidar() -> Workload:
    ss = np.random.SeedSequence(SEEDS["lidar"]).spawn(8)
    r_layout, r_noise1, r_noise2, r_out1, r_out2, _, _, _ = [np.random.Generator(np.random.PCG64(s)) for s in ss]
    cx = r_layout.uniform(-40, 40, 40)
    cy = r_layout.uniform(5.5, 7.5, 40) * np.where(r_layout.uniform(size=40) < 0.5, -1.0, 1.0)
    cyl = list(zip(cx, cy))
    h = 1.73
    R1 = np.eye(3)
    c1 = np.array([0.0, 0.0, h])
    R2 = _rot_z(np.deg2rad(5.0))
    c2 = np.array([1.0, 0.0, h])
    P1 = _lidar_scan(r_noise1, R1, c1, cyl)
    P2 = _lidar_scan(r_noise2, R2, c2, cyl)
    n_hits = (P1.shape[0], P2.shape[0])
    Y, inl_y = _add_uniform_outliers(r_out1, P1, 0.10, lo=np.full(3, -50.0), hi=np.full(3, 50.0))
    X, inl_x = _add_uniform_outliers(r_out2, P2, 0.10, lo=np.full(3, -50.0), hi=np.full(3, 50.0))
    R_e = R1.T @ R2
    t_e = R1.T @ (c2 - c1)
    return Workload("lidar", _f32(Y), _f32(X), R_e, t_e, 0.1, 50, 10, inl_y, inl_x,
                    {"seed": SEEDS["lidar"], "hits": n_hits, "rings": 64, "azimuths": 1800,
                     "elev_deg": [2.0, -24.8], "height": h, "facade_y": 8.0, "facade_h": 12.0,
                     "cylinders": 40, "cyl_r": 0.15, "cyl_h": 4.0, "range_noise": 0.02, "max_range": 120.0,
                     "outlier_box": [-50, 50], "outlier_frac": 0.10, "motion": "1 m forward, 5 deg yaw"})


def make_scale(n: int = 524288) -> Workload:
    ss = np.random.SeedSequence(SEEDS["scale"]).spawn(8)
    r_layout, r_tgt, r_src, r_noise, r_axis, r_dir, _, _ = [np.random.Generator(np.random.PCG64(s)) for s in ss]
    layout_state = r_layout.bit_generator.state
    Y = sample_patches_spheres(r_layout, r_tgt, n)
    r_layout.bit_generator.state = layout_state            # same layout for the source resample
    Xs = sample_patches_spheres(r_layout, r_src, n)
    Y = Y + r_noise.standard_normal(Y.shape) * 0.002
    Xs = Xs + r_noise.standard_normal(Xs.shape) * 0.002
    R_gt = axis_angle(_unit(r_axis), np.deg2rad(60.0))
    t_gt = 0.3 * _unit(r_dir)
    X = _apply(R_gt, t_gt, Xs)
    R_e, t_e = _inverse(R_gt, t_gt)
    return Workload("scale", _f32(Y), _f32(X), R_e, t_e, 0.2, 30, 10, np.ones(n, bool), np.ones(n, bool),
                    {"seed": SEEDS["scale"], "patches": 64, "spheres": 64, "noise_sd": 0.002,
                     "rot_deg": 60.0, "t_norm": 0.3})


def sample_desk_scene(rng: np.random.Generator, n: int, radii, centers) -> np.ndarray:
    """Desk corner: floor [-0.5,0.5]² at z = 0, walls x = -0.5 and y = -0.5 of height 0.5, plus upper
    hemispheres of `radii` at `centers` (on the floor), area-proportional (SPEC S:630's desk-scale plane +
    hemisphere, with walls and a second hemisphere so that no rotation maps the scene onto itself)."""
    areas = np.array([1.0, 0.5, 0.5] + [2.0 * np.pi * r * r for r in radii])
    counts = rng.multinomial(n, areas / areas.sum())
    P = np.empty((n, 3))
    k0, k1, k2 = counts[:3]
    P[:k0, 0:2] = rng.uniform(-0.5, 0.5, (k0, 2))                     # floor z = 0
    P[:k0, 2] = 0.0
    P[k0:k0 + k1, 0] = -0.5                                            # wall x = -0.5, height 0.5
    P[k0:k0 + k1, 1] = rng.uniform(-0.5, 0.5, k1)
    P[k0:k0 + k1, 2] = rng.uniform(0.0, 0.5, k1)
    P[k0 + k1:k0 + k1 + k2, 1] = -0.5                                  # wall y = -0.5
    P[k0 + k1:k0 + k1 + k2, 0] = rng.uniform(-0.5, 0.5, k2)
    P[k0 + k1:k0 + k1 + k2, 2] = rng.uniform(0.0, 0.5, k2)
    o = k0 + k1 + k2
    for r, c, k in zip(radii, centers, counts[3:]):
        d = rng.standard_normal((k, 3))
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        d[:, 2] = np.abs(d[:, 2])
        P[o:o + k] = np.asarray(c) + r * d
        o += k
    return P


BATCH_SEED = 6


def make_batch(B: int = 550, n: int = 3500, seed: int = BATCH_SEED, ragged: bool = False):
    """Many small registration problems (the paper's problem size: 3.5k-5k points,
    P:359-360): problem b is a desk scene (plane + hemisphere of radius U(0.2, 0.35) at a
    random spot) with noise sd 0.005, an independent resample for the source, rotated 50° about a random
    axis (the §4.1 protocol) and translated by 0.1·random unit vector; w = 0.1, 50 EM iterations.
    ragged: sizes vary per problem (n/2 .. 3n/2).  Returns a list of Workloads."""
    out = []
    ss = np.random.SeedSequence(seed).spawn(B)
    for b in range(B):
        r_lay, r_t, r_s, r_noise, r_axis, r_dir, r_n = [np.random.Generator(np.random.PCG64(s)) for s in ss[b].spawn(7)]
        rad = [r_lay.uniform(0.15, 0.25), r_lay.uniform(0.06, 0.1)]
        ang = r_lay.uniform(0, 2 * np.pi)
        c = [np.array([0.2 * np.cos(ang), 0.2 * np.sin(ang), 0.0]), np.array([-0.3 * np.cos(ang), -0.3 * np.sin(ang), 0.0])]
        nm = int(r_n.integers(n // 2, 3 * n // 2 + 1)) if ragged else n
        ns = int(r_n.integers(n // 2, 3 * n // 2 + 1)) if ragged else n
        Y = sample_desk_scene(r_t, nm, rad, c) + r_noise.standard_normal((nm, 3)) * 0.005
        Xs = sample_desk_scene(r_s, ns, rad, c) + r_noise.standard_normal((ns, 3)) * 0.005
        R_gt = axis_angle(_unit(r_axis), np.deg2rad(50.0))
        t_gt = 0.1 * _unit(r_dir)
        X = _apply(R_gt, t_gt, Xs)
        R_e, t_e = _inverse(R_gt, t_gt)
        out.append(Workload(f"batch{b}", _f32(Y), _f32(X), R_e, t_e, 0.1, 50, 10, np.ones(nm, bool),
                            np.ones(ns, bool), {"seed": seed, "index": b, "radii": rad, "rot_deg": 50.0,
                                                "t_norm": 0.1, "noise_sd": 0.005}))
    return out


def make(name: str) -> Workload:
    if name == "tiny":
        return make_tiny()
    if name == "tiny_noiseless":
        return make_tiny(noiseless=True)
    if name == "object":
        return make_object()
    if name == "object_noiseless":
        return make_object(noiseless=True)
    if name == "rgbd":
        return make_rgbd()
    if name == "lidar":
        return make_lidar()
    if name == "scale":
        return make_scale()
    raise KeyError(name)


def random_rigid(rng: np.random.Generator, max_angle_deg: float, t_scale: float):
    """A random rigid motion (test helper): axis uniform, angle U(0, max), t Gaussian·scale."""
    R = axis_angle(_unit(rng), np.deg2rad(rng.uniform(0, max_angle_deg)))
    t = rng.standard_normal(3) * t_scale
    return R, t
