"""Seeded synthetic inputs for the FEC hot path (shared by the oracle side and the CUDA side).

This module only *makes point clouds*: it holds none of the clustering arithmetic
(no distance predicate, no grid, no union-find).  Both `oracle/` and the CUDA
binding consume the arrays it returns; neither imports the other.

Every generator uses numpy PCG64 (`default_rng(seed)`), does its geometry in
float64 and casts to float32 at the end, row-major ``[n, 3]``.

Workloads (BASELINE.json ``configs``; concrete recipe in SURVEY.md §8(d) and DESIGN.md §3):

* ``C1`` — 20 Gaussian blobs (sigma 0.3 m, 400 pts) + 2,000 uniform noise points in
  [0,50]^3, shuffled (the paper's "unorganized" index order, §3.3.1).
* ``C2`` — one synthetic 64-beam spinning-LiDAR scan, ground removed (stands in for a
  single KITTI scan, Table 4; KITTI itself is not available).
* ``C3`` — 100 such scans accumulated along a gently curving path (stands in for the
  accumulated KITTI sequences of Table 2).
* ``C4`` — a 27M-point accumulated loop map (Fig. 1 "27 million points").
* ``C5`` — 100M uniform points at mean degree 2.8 (near continuum percolation; density
  from nu = 4/3 pi d^3 rho) + 50 dense balls, shuffled.
"""
from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass

import numpy as np

__all__ = [
    "Workload", "CONFIGS", "make_config", "c1_blobs", "lidar_scan", "c3_map", "c4_loop",
    "c5_stress", "random_cloud", "PARITY_GEOMETRIES", "sha256_f32", "lidar_scan_ground", "ground_map",
    "plane_and_box", "ransac_triplets", "make_ground_config", "GROUND_PARAMS", "voxel_clusters",
]


@dataclass
class Workload:
    name: str
    points: np.ndarray          # float32 [n, 3], C-contiguous
    d_th: float
    min_size: int
    max_size: int
    meta: dict

    @property
    def n(self) -> int:
        return int(self.points.shape[0])


def sha256_f32(points: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(points, dtype=np.float32).tobytes()).hexdigest()


def _f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


# --------------------------------------------------------------------------------------
# C1: blobs + noise
# --------------------------------------------------------------------------------------
def c1_blobs(seed: int = 0, n_blobs: int = 20, per_blob: int = 400, n_noise: int = 2000,
             box: float = 50.0, sigma: float = 0.3) -> np.ndarray:
    rng = np.random.default_rng(seed)
    centres = rng.uniform(0.0, box, size=(n_blobs, 3))
    blobs = centres[:, None, :] + rng.normal(0.0, sigma, size=(n_blobs, per_blob, 3))
    noise = rng.uniform(0.0, box, size=(n_noise, 3))
    pts = np.concatenate([blobs.reshape(-1, 3), noise], axis=0)
    perm = rng.permutation(pts.shape[0])
    return _f32(pts[perm])


# --------------------------------------------------------------------------------------
# LiDAR ray caster (C2/C3/C4).  Geometry only: nearest ray/solid intersection.
# --------------------------------------------------------------------------------------
SENSOR_H = 1.73
N_RINGS = 64
N_AZ = 2048
ELEV = np.deg2rad(np.linspace(-24.8, 2.0, N_RINGS))
BOX_L, BOX_W, BOX_H = 4.0, 1.8, 1.5
CYL_R, CYL_H = 0.15, 3.0
MAX_RANGE = 120.0
BOX_RHO = math.hypot(BOX_L / 2, BOX_W / 2)


def _column_pairs(rel_x, rel_y, rho, yaw):
    """For objects at sensor-relative xy, return (obj_id, column) pairs whose azimuth
    column can intersect the object's bounding circle of radius ``rho``."""
    r = np.hypot(rel_x, rel_y)
    bearing = np.arctan2(rel_y, rel_x) - yaw
    half = np.where(r > rho, np.arcsin(np.minimum(rho / np.maximum(r, 1e-12), 1.0)), np.pi)
    step = 2 * np.pi / N_AZ
    lo = np.floor((bearing - half) / step).astype(np.int64) - 1
    hi = np.ceil((bearing + half) / step).astype(np.int64) + 1
    cnt = np.minimum(hi - lo + 1, N_AZ)
    obj = np.repeat(np.arange(rel_x.shape[0]), cnt)
    start = np.repeat(lo, cnt)
    offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
    col = np.mod(start + offs, N_AZ)
    return obj, col


def _ray_dirs(yaw: float, cols: np.ndarray):
    """World-frame unit directions for all 64 rings of the given azimuth columns.
    Returns arrays shaped [len(cols), 64]."""
    az = cols.astype(np.float64) * (2 * np.pi / N_AZ) + yaw
    ce, se = np.cos(ELEV), np.sin(ELEV)
    dx = np.cos(az)[:, None] * ce[None, :]
    dy = np.sin(az)[:, None] * ce[None, :]
    dz = np.broadcast_to(se[None, :], dx.shape)
    return dx, dy, dz


def _cast_boxes(ox, oy, boxes, t_best, yaw):
    """boxes: [k, 3] (cx, cy, byaw).  Updates t_best[N_AZ, N_RINGS] in place."""
    if boxes.shape[0] == 0:
        return
    obj, col = _column_pairs(boxes[:, 0] - ox, boxes[:, 1] - oy, BOX_RHO, yaw)
    dx, dy, dz = _ray_dirs(yaw, col)
    cx, cy, by = boxes[obj, 0][:, None], boxes[obj, 1][:, None], boxes[obj, 2][:, None]
    cb, sb = np.cos(by), np.sin(by)
    # ray origin / direction in the box frame (rotate by -byaw about z)
    rx, ry = ox - cx, oy - cy
    lox, loy = cb * rx + sb * ry, -sb * rx + cb * ry
    ldx, ldy = cb * dx + sb * dy, -sb * dx + cb * dy
    with np.errstate(divide="ignore", invalid="ignore"):
        tx1 = (-BOX_L / 2 - lox) / ldx
        tx2 = (BOX_L / 2 - lox) / ldx
        ty1 = (-BOX_W / 2 - loy) / ldy
        ty2 = (BOX_W / 2 - loy) / ldy
        tz1 = (0.0 - SENSOR_H) / dz
        tz2 = (BOX_H - SENSOR_H) / dz
        tn = np.maximum(np.maximum(np.minimum(tx1, tx2), np.minimum(ty1, ty2)), np.minimum(tz1, tz2))
        tf = np.minimum(np.minimum(np.maximum(tx1, tx2), np.maximum(ty1, ty2)), np.maximum(tz1, tz2))
        hit = (tn <= tf) & (tn > 0) & np.isfinite(tn)
    t = np.where(hit, tn, np.inf)
    colb = np.broadcast_to(col[:, None], t.shape)
    ring = np.broadcast_to(np.arange(N_RINGS)[None, :], t.shape)
    np.minimum.at(t_best, (colb.ravel(), ring.ravel()), t.ravel())


def _cast_cyls(ox, oy, cyls, t_best, yaw):
    """cyls: [k, 2] (cx, cy)."""
    if cyls.shape[0] == 0:
        return
    obj, col = _column_pairs(cyls[:, 0] - ox, cyls[:, 1] - oy, CYL_R, yaw)
    dx, dy, dz = _ray_dirs(yaw, col)
    rx = (ox - cyls[obj, 0])[:, None]
    ry = (oy - cyls[obj, 1])[:, None]
    a = dx * dx + dy * dy
    b = 2.0 * (rx * dx + ry * dy)
    c = rx * rx + ry * ry - CYL_R * CYL_R
    disc = b * b - 4.0 * a * c
    with np.errstate(invalid="ignore", divide="ignore"):
        tn = (-b - np.sqrt(disc)) / (2.0 * a)
        z = SENSOR_H + tn * dz
        hit = (disc >= 0) & (tn > 0) & (z >= 0.0) & (z <= CYL_H)
    t = np.where(hit, tn, np.inf)
    colb = np.broadcast_to(col[:, None], t.shape)
    ring = np.broadcast_to(np.arange(N_RINGS)[None, :], t.shape)
    np.minimum.at(t_best, (colb.ravel(), ring.ravel()), t.ravel())


def _scan(rng, ox, oy, yaw, boxes, cyls, noise_sigma=0.02, keep_ground=False):
    """One spinning scan from sensor (ox, oy, SENSOR_H) with heading ``yaw``.
    Returns float64 [m, 3] object hits in azimuth-major acquisition order (plus the hits
    on the ground plane z = 0 when ``keep_ground``)."""
    t_best = np.full((N_AZ, N_RINGS), np.inf)
    _cast_boxes(ox, oy, boxes, t_best, yaw)
    _cast_cyls(ox, oy, cyls, t_best, yaw)
    se = np.sin(ELEV)
    with np.errstate(divide="ignore"):
        t_ground = np.where(se < 0, -SENSOR_H / se, np.inf)[None, :]
    if keep_ground:
        t_best = np.minimum(t_best, t_ground)
    keep = (t_best < t_ground) & (t_best <= MAX_RANGE)
    if keep_ground:
        keep = t_best <= MAX_RANGE
    # range noise is drawn for every ray so the RNG stream does not depend on hits
    noise = rng.normal(0.0, noise_sigma, size=t_best.shape)
    cols, rings = np.nonzero(keep)          # row-major => azimuth-major order
    t = t_best[cols, rings] + noise[cols, rings]
    az = cols * (2 * np.pi / N_AZ) + yaw
    ce = np.cos(ELEV[rings])
    pts = np.empty((t.shape[0], 3))
    pts[:, 0] = ox + t * ce * np.cos(az)
    pts[:, 1] = oy + t * ce * np.sin(az)
    pts[:, 2] = SENSOR_H + t * np.sin(ELEV[rings])
    return pts


def _objects_around(rng, ox, oy, n_boxes, n_cyls, r_lo=5.0, r_hi=60.0):
    def place(k):
        r = rng.uniform(r_lo, r_hi, size=k)
        th = rng.uniform(0.0, 2 * np.pi, size=k)
        return ox + r * np.cos(th), oy + r * np.sin(th)
    bx, by = place(n_boxes)
    byaw = rng.uniform(0.0, np.pi, size=n_boxes)
    cx, cy = place(n_cyls)
    return np.stack([bx, by, byaw], 1), np.stack([cx, cy], 1)


def lidar_scan(seed: int = 1, n_boxes: int = 60, n_cyls: int = 40) -> np.ndarray:
    """C2: one 64-beam scan from (0, 0, 1.73), ground hits removed."""
    rng = np.random.default_rng(seed)
    boxes, cyls = _objects_around(rng, 0.0, 0.0, n_boxes, n_cyls)
    return _f32(_scan(rng, 0.0, 0.0, 0.0, boxes, cyls))


def c3_map(seed: int = 2, n_poses: int = 100, n_boxes: int = 300, n_cyls: int = 200,
           yaw_step_deg: float = 0.5, step_m: float = 1.0) -> np.ndarray:
    """C3: scans accumulated along a gently curving path; every scan has its own objects."""
    rng = np.random.default_rng(seed)
    x = y = yaw = 0.0
    out = []
    for k in range(n_poses):
        if k > 0:
            yaw += math.radians(yaw_step_deg)
            x += step_m * math.cos(yaw)
            y += step_m * math.sin(yaw)
        boxes, cyls = _objects_around(rng, x, y, n_boxes, n_cyls)
        out.append(_scan(rng, x, y, yaw, boxes, cyls))
    return _f32(np.concatenate(out, 0))


# --------------------------------------------------------------------------------------
# Ground-removal inputs: scans WITH their ground hits, tilted as a whole
# (a pitched sensor / sloped road), and the caller-drawn RANSAC index triplets.
# --------------------------------------------------------------------------------------
GROUND_PARAMS = {"threshold": 0.2, "iterations": 100, "max_tilt_deg": 30.0}  # SPEC.md L323 defaults


def _tilt(pts: np.ndarray, tilt_deg: float, axis_deg: float = 30.0) -> np.ndarray:
    """Rotate by ``tilt_deg`` about the horizontal axis at bearing ``axis_deg``."""
    a = math.radians(axis_deg)
    k = np.array([math.cos(a), math.sin(a), 0.0])
    t = math.radians(tilt_deg)
    K = np.array([[0, -k[2], k[1]], [k[2], 0, -k[0]], [-k[1], k[0], 0]])
    R = np.eye(3) + math.sin(t) * K + (1 - math.cos(t)) * (K @ K)
    return pts @ R.T


def lidar_scan_ground(seed: int = 5, n_boxes: int = 60, n_cyls: int = 40, tilt_deg: float = 2.0) -> np.ndarray:
    """G2: one 64-beam scan with its ground hits kept (~75% of the points), tilted."""
    rng = np.random.default_rng(seed)
    boxes, cyls = _objects_around(rng, 0.0, 0.0, n_boxes, n_cyls)
    return _f32(_tilt(_scan(rng, 0.0, 0.0, 0.0, boxes, cyls, keep_ground=True), tilt_deg))


def ground_map(seed: int = 6, n_poses: int = 100, n_boxes: int = 300, n_cyls: int = 200,
               tilt_deg: float = 2.0) -> np.ndarray:
    """G3: C3's recipe (scans along a gently curving path) with the ground hits kept."""
    rng = np.random.default_rng(seed)
    x = y = yaw = 0.0
    out = []
    for k in range(n_poses):
        if k > 0:
            yaw += math.radians(0.5)
            x += math.cos(yaw)
            y += math.sin(yaw)
        boxes, cyls = _objects_around(rng, x, y, n_boxes, n_cyls)
        out.append(_scan(rng, x, y, yaw, boxes, cyls, keep_ground=True))
    return _f32(_tilt(np.concatenate(out, 0), tilt_deg))


def plane_and_box(seed: int = 7, n_plane: int = 1000, n_box: int = 100) -> np.ndarray:
    """SPEC.md L313's example: n_plane points on z = 0 then n_box points in a box at z in [1, 3]."""
    rng = np.random.default_rng(seed)
    g = np.zeros((n_plane, 3))
    g[:, :2] = rng.uniform(-10.0, 10.0, size=(n_plane, 2))
    b = rng.uniform([2.0, 2.0, 1.0], [4.0, 4.0, 3.0], size=(n_box, 3))
    return _f32(np.concatenate([g, b], 0))


def ransac_triplets(n: int, H: int = 100, seed: int = 0) -> np.ndarray:
    """int32 [H, 3]: per hypothesis three distinct indices in [0, n) (the random sample a
    RANSAC iteration draws, passed to both the oracle and the CUDA path; reading G1)."""
    rng = np.random.default_rng(10_000 + seed)
    if n < 3:
        return rng.integers(0, max(n, 1), size=(H, 3)).astype(np.int32)
    t = rng.integers(0, n, size=(H, 3))
    for _ in range(100):
        bad = (t[:, 0] == t[:, 1]) | (t[:, 0] == t[:, 2]) | (t[:, 1] == t[:, 2])
        if not bad.any():
            break
        t[bad] = rng.integers(0, n, size=(int(bad.sum()), 3))
    return np.ascontiguousarray(t, dtype=np.int32)


def make_ground_config(name: str, scale: float = 1.0):
    """(points, triplets, threshold, max_tilt_deg) for G2 / G3 (scale shrinks G3's poses)."""
    if name == "G2":
        pts = lidar_scan_ground(5)
    elif name == "G3":
        pts = ground_map(6, n_poses=max(1, int(round(100 * scale))))
    else:
        raise KeyError(name)
    H = GROUND_PARAMS["iterations"]
    return pts, ransac_triplets(pts.shape[0], H, seed=int(name[1:])), GROUND_PARAMS["threshold"], \
        GROUND_PARAMS["max_tilt_deg"]


# --------------------------------------------------------------------------------------
# Voxel-fill clusters with ground truth (§3.3.1): the
# synthetic setting of the paper's Fig. 4-6, for the AP metric.
# --------------------------------------------------------------------------------------
def voxel_clusters(n_clusters: int, density: int, voxel_edge: float = 1.0, shift_sigma: float = 0.0,
                   seed: int = 0):
    """(points float32 [n*m, 3], gt int32 labels 1..n, recommended d_th).

    n voxels on a stride-2 lattice (>= one voxel edge of empty space between any two), each
    filled with the first m sites (lexicographic) of an even g^3 grid, g = ceil(m^(1/3)),
    pitch = edge/(g-1); optional normal shift clamped to the voxel; shuffled point order."""
    rng = np.random.default_rng(seed)
    g = max(1, int(math.ceil(round(density ** (1.0 / 3.0), 9))))
    while g ** 3 < density:
        g += 1
    pitch = voxel_edge / (g - 1) if g > 1 else 0.0
    d_th = 1.1 * pitch if g > 1 else 0.5 * voxel_edge
    if d_th >= voxel_edge:
        raise ValueError("density too low for the separation guarantee (recommended d_th >= voxel edge)")
    side = int(math.ceil(n_clusters ** (1.0 / 3.0))) + 1
    while side ** 3 < n_clusters:
        side += 1
    cells = rng.choice(side ** 3, size=n_clusters, replace=False)
    lat = np.stack([cells % side, (cells // side) % side, cells // (side * side)], 1).astype(np.float64)
    origin = lat * (2.0 * voxel_edge)
    sites = np.stack(np.meshgrid(np.arange(g), np.arange(g), np.arange(g), indexing="ij"), -1).reshape(-1, 3)
    sites = sites[:density].astype(np.float64) * pitch if g > 1 else np.full((1, 3), 0.5 * voxel_edge)
    pts = (origin[:, None, :] + sites[None, :, :]).reshape(-1, 3)
    gt = np.repeat(np.arange(1, n_clusters + 1, dtype=np.int32), sites.shape[0])
    if shift_sigma > 0:
        lo = np.repeat(origin, sites.shape[0], axis=0)
        pts = np.clip(pts + rng.normal(0.0, shift_sigma, size=pts.shape), lo, lo + voxel_edge)
    perm = rng.permutation(pts.shape[0])
    return _f32(pts[perm]), np.ascontiguousarray(gt[perm]), float(np.float32(d_th))


C4_LATERAL_HI = 6.5


def c4_loop(seed: int = 3, n_poses: int = 450, n_boxes: int = 1200, n_cyls: int = 800,
            circumference: float = 2000.0, lateral=(2.0, C4_LATERAL_HI),
            pose_range: tuple | None = None) -> np.ndarray:
    """C4: a 2 km circular loop map, static roadside objects, 450 poses.

    ``pose_range=(a, b)`` casts only poses a..b-1 (same objects, same RNG stream per
    pose) -- used for scaled-down test slices."""
    rng = np.random.default_rng(seed)
    R = circumference / (2 * np.pi)

    def roadside(k):
        s = rng.uniform(0.0, circumference, size=k)
        lat = rng.uniform(lateral[0], lateral[1], size=k) * np.where(rng.random(k) < 0.5, -1.0, 1.0)
        ang = s / R
        rr = R + lat
        return rr * np.cos(ang), rr * np.sin(ang)

    bx, by = roadside(n_boxes)
    byaw = rng.uniform(0.0, np.pi, size=n_boxes)
    cx, cy = roadside(n_cyls)
    # resample any box footprint reaching within 1 m of the centreline
    for _ in range(100):
        dist = np.abs(np.hypot(bx, by) - R)
        bad = dist < 1.0 + BOX_RHO
        if not bad.any():
            break
        nbx, nby = roadside(int(bad.sum()))
        bx[bad], by[bad] = nbx, nby
    boxes = np.stack([bx, by, byaw], 1)
    cyls = np.stack([cx, cy], 1)
    seeds = rng.integers(0, 2**63 - 1, size=n_poses)
    a, b = pose_range if pose_range is not None else (0, n_poses)
    out = []
    for k in range(a, b):
        ang = 2 * np.pi * k / n_poses
        ox, oy = R * math.cos(ang), R * math.sin(ang)
        yaw = ang + np.pi / 2
        near_b = np.hypot(boxes[:, 0] - ox, boxes[:, 1] - oy) < 125.0
        near_c = np.hypot(cyls[:, 0] - ox, cyls[:, 1] - oy) < 125.0
        prng = np.random.default_rng(int(seeds[k]))
        out.append(_scan(prng, ox, oy, yaw, boxes[near_b], cyls[near_c]))
    return _f32(np.concatenate(out, 0))


C5_NU = 2.8
C5_D = 0.1


def c5_side(n_uniform: int, d: float = C5_D, nu: float = C5_NU) -> float:
    """Cube side so that the mean neighbour count within d is nu (nu = 4/3 pi d^3 rho)."""
    return (n_uniform * (4.0 / 3.0) * math.pi * d ** 3 / nu) ** (1.0 / 3.0)


def c5_stress(seed: int = 4, n_uniform: int = 100_000_000, n_balls: int = 50,
              ball_pts: int = 200_000, ball_r: float = 0.2, chunk: int = 10_000_000) -> np.ndarray:
    rng = np.random.default_rng(seed)
    L = c5_side(n_uniform)
    n = n_uniform + n_balls * ball_pts
    pts = np.empty((n, 3), dtype=np.float32)
    for s in range(0, n_uniform, chunk):
        e = min(n_uniform, s + chunk)
        pts[s:e] = rng.uniform(0.0, L, size=(e - s, 3))
    centres = rng.uniform(ball_r, L - ball_r, size=(n_balls, 3))
    off = n_uniform
    for k in range(n_balls):
        r = ball_r * rng.random(ball_pts) ** (1.0 / 3.0)
        v = rng.normal(size=(ball_pts, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        pts[off:off + ball_pts] = centres[k] + r[:, None] * v
        off += ball_pts
    perm = rng.permutation(n)
    return np.ascontiguousarray(pts[perm])


CONFIGS = {
    # name: (d_th, min_size, max_size)
    "C1": (0.5, 10, 1_000_000),
    "C2": (0.35, 50, 25_000),
    "C3": (0.2, 50, 1_000_000),
    "C4": (0.25, 100, 5_000_000),
    "C5": (0.1, 1, 1_000_000_000),
}


def make_config(name: str, scale: float = 1.0) -> Workload:
    """Build a BASELINE.json config.  ``scale < 1`` shrinks C3/C4/C5 for tests while
    keeping their densities (fewer poses / fewer points in a proportionally smaller cube)."""
    d_th, mn, mx = CONFIGS[name]
    meta = {"scale": scale}
    if name == "C1":
        pts = c1_blobs(0)
    elif name == "C2":
        pts = lidar_scan(1)
    elif name == "C3":
        pts = c3_map(2, n_poses=max(1, int(round(100 * scale))))
    elif name == "C4":
        n_poses = 450
        if scale < 1.0:
            k = max(1, int(round(n_poses * scale)))
            pts = c4_loop(3, pose_range=(0, k))
        else:
            pts = c4_loop(3)
    elif name == "C5":
        nu = max(1000, int(round(100_000_000 * scale)))
        bp = max(100, int(round(200_000 * scale)))
        pts = c5_stress(4, n_uniform=nu, ball_pts=bp)
        meta["side_m"] = c5_side(nu)
    else:
        raise KeyError(name)
    return Workload(name, pts, d_th, mn, mx, meta)


# --------------------------------------------------------------------------------------
# Small random parity clouds (T2/T5 sets): mixed geometries that stress boundaries.
# --------------------------------------------------------------------------------------
PARITY_GEOMETRIES = ("uniform", "blobs", "duplicates", "line", "lattice", "cell_edges", "mixed")


def random_cloud(seed: int, n: int | None = None, geometry: str | None = None):
    """Returns (points float32 [n,3], d_th float32-representable float, geometry)."""
    rng = np.random.default_rng(1000 + seed)
    if geometry is None:
        geometry = PARITY_GEOMETRIES[seed % len(PARITY_GEOMETRIES)]
    if n is None:
        n = int(rng.integers(1, 2001))
    d = float(np.float32(rng.uniform(0.05, 2.0)))
    if geometry == "uniform":
        side = float(rng.uniform(1.0, 30.0))
        p = rng.uniform(-side / 2, side / 2, size=(n, 3)) + rng.uniform(-100, 100, size=3)
    elif geometry == "blobs":
        k = int(rng.integers(1, 12))
        c = rng.uniform(0, 20, size=(k, 3))
        p = c[rng.integers(0, k, size=n)] + rng.normal(0, rng.uniform(0.05, 1.0), size=(n, 3))
    elif geometry == "duplicates":
        m = max(1, n // 4)
        base = rng.uniform(0, 5, size=(m, 3))
        p = base[rng.integers(0, m, size=n)]
    elif geometry == "line":
        t = rng.uniform(0, 1, size=n) * n * d * float(rng.uniform(0.3, 1.5))
        dirv = rng.normal(size=3)
        dirv /= np.linalg.norm(dirv)
        p = t[:, None] * dirv[None, :]
    elif geometry == "lattice":
        # dyadic spacing => exact fp32 coordinates and exact squared distances
        d = float(rng.choice([0.25, 0.5, 1.0, 2.0]))
        sp = d * float(rng.choice([0.5, 1.0, 1.0, 1.5]))
        side = max(1, int(round(n ** (1 / 3))) + 1)
        g = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
        g = g[rng.permutation(g.shape[0])[:n]]
        p = g * sp + float(rng.integers(-8, 8)) * 4.0
    elif geometry == "cell_edges":
        # points exactly d apart along axes and at multiples of d (worst case for grids)
        d = float(rng.choice([0.125, 0.5, 1.0, 3.0]))
        k = rng.integers(-6, 7, size=(n, 3)).astype(np.float64)
        jitter = rng.integers(0, 2, size=(n, 3)) * np.float64(np.spacing(np.float32(d)))
        p = k * d + jitter
    else:  # mixed
        parts = [rng.uniform(0, 10, size=(n // 2, 3)),
                 rng.normal(5, 0.2, size=(n - n // 2, 3))]
        p = np.concatenate(parts, 0)[rng.permutation(n)]
    return _f32(p), d, geometry
