"""Ground-removal oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

RANSAC plane fit with a vertical-tilt constraint, then least-squares refinement, then
removal of the inliers: SPEC.md L307-310 (op ``remove_ground``), the pre-processing step
of PAPER.md L179-184 (§2.1).  The per-hypothesis arithmetic (plane, residual, inlier test)
is plain C in ground_oracle.c; this module follows SPEC's steps in order:

1. hypotheses: the caller's index triplets (reading G1), one plane each (G2);
2. count the inliers of every plane (G3);
3. keep the best tilt-valid plane, the lowest index among equal counts (G4);
4. ground iff that count >= min_inliers (SPEC: ">= 10% inliers"; G5);
5. refine by least squares over its inliers: centroid + the eigenvector of the smallest
   eigenvalue of the scatter matrix (numpy.linalg.eigh as the library step), oriented
   n_z >= 0, offset = -n . centroid (G7);
6. remove the inliers of the best hypothesis plane, survivors in input order (G6).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import lib, _pts


@dataclass
class GroundResult:
    best: int                 # hypothesis index, -1 = no ground
    n_inliers: int            # inliers of the best plane (0 when no ground)
    plane: np.ndarray         # float32 [4] (nx, ny, nz, off) of the best hypothesis (NaN: none)
    refined: np.ndarray       # float64 [4] least-squares plane over its inliers (NaN: none)
    counts: np.ndarray        # int64 [H] inliers of every hypothesis plane (0: no plane)
    valid: np.ndarray         # int32 [H] plane exists and is within the tilt bound
    planes: np.ndarray        # float32 [H, 4]
    ground: np.ndarray        # bool [n] removed points
    keep_idx: np.ndarray      # int32 [n_keep] survivors' input indices, increasing
    keep_points: np.ndarray   # float32 [n_keep, 3]


def plane(points, triplet, cos_max_tilt: float):
    """(exists, tilt_ok, float32[4]) for one hypothesis (G2)."""
    p = _pts(points)
    t = np.ascontiguousarray(triplet, dtype=np.int32)
    out = np.zeros(4, dtype=np.float32)
    ok = ctypes.c_int32(0)
    ex = lib().oracle_ground_plane(p.ctypes.data, p.shape[0], t.ctypes.data, float(cos_max_tilt),
                                   out.ctypes.data, ctypes.byref(ok))
    return bool(ex), bool(ok.value), out


def residual(plane_f32, p) -> np.float32:
    pl = np.ascontiguousarray(plane_f32, dtype=np.float32)
    q = np.ascontiguousarray(p, dtype=np.float32)
    return np.float32(lib().oracle_ground_residual(pl.ctypes.data, q.ctypes.data))


def counts(points, triplets, threshold: float, cos_max_tilt: float):
    p = _pts(points)
    t = np.ascontiguousarray(triplets, dtype=np.int32).reshape(-1, 3)
    H = t.shape[0]
    planes = np.zeros((H, 4), dtype=np.float32)
    valid = np.zeros(H, dtype=np.int32)
    cnt = np.zeros(H, dtype=np.int64)
    lib().oracle_ground_counts(p.ctypes.data, p.shape[0], t.ctypes.data, H, ctypes.c_float(np.float32(threshold)),
                               float(cos_max_tilt), planes.ctypes.data, valid.ctypes.data, cnt.ctypes.data)
    return planes, valid, cnt


def inlier_mask(points, plane_f32, threshold: float) -> np.ndarray:
    p = _pts(points)
    pl = np.ascontiguousarray(plane_f32, dtype=np.float32)
    m = np.zeros(p.shape[0], dtype=np.uint8)
    lib().oracle_ground_mask(p.ctypes.data, p.shape[0], pl.ctypes.data, ctypes.c_float(np.float32(threshold)),
                             m.ctypes.data)
    return m.astype(bool)


def refine(inlier_points) -> np.ndarray:
    """Least-squares plane through the points (step 5, reading G7): float64 (nx, ny, nz, off)."""
    q = np.asarray(inlier_points, dtype=np.float64)
    c = q.mean(axis=0)
    d = q - c
    scatter = d.T @ d
    _, vecs = np.linalg.eigh(scatter)   # ascending eigenvalues
    nrm = vecs[:, 0]
    if nrm[2] < 0:
        nrm = -nrm
    return np.array([nrm[0], nrm[1], nrm[2], -float(nrm @ c)])


def ransac_ground(points, triplets, threshold: float, cos_max_tilt: float, min_inliers: int) -> GroundResult:
    p = _pts(points)
    n = p.shape[0]
    planes, valid, cnt = counts(p, triplets, threshold, cos_max_tilt)
    best = -1
    for h in range(planes.shape[0]):           # step 3: first strict maximum among valid
        if valid[h] and (best < 0 or cnt[h] > cnt[best]):
            best = h
    if best >= 0 and cnt[best] < int(min_inliers):
        best = -1
    nan4 = np.full(4, np.nan)
    if best < 0:
        return GroundResult(-1, 0, nan4.astype(np.float32), nan4, cnt, valid, planes, np.zeros(n, bool),
                            np.arange(n, dtype=np.int32), p.copy())
    ground = inlier_mask(p, planes[best], threshold)
    assert int(ground.sum()) == int(cnt[best])
    refined = refine(p[ground]) if ground.sum() >= 3 else planes[best].astype(np.float64)
    keep = np.nonzero(~ground)[0].astype(np.int32)
    return GroundResult(best, int(cnt[best]), planes[best].copy(), refined, cnt, valid, planes, ground, keep,
                        p[keep].copy())
