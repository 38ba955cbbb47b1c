"""FEC oracle, brute-force form — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The definition written out, O(n^2), numpy float32 (numpy evaluates every float32
operation with one IEEE round-to-nearest and never contracts to FMA):

  pred(i,j): d2 = ((dx*dx + dy*dy) + dz*dz) <= t2,  dx = x_j - x_i, ...,  t2 = fl32(d*d)
             -- PAPER.md L187-194 (Eq. 1), readings A1-A3.
  labels[i] = min C(i)                        -- the component of i, canonicalised to its
                                                 smallest index (reading A8)
  labels[i] = -1 if |C(i)| outside [min_size, max_size]   (readings A7, A10)

min C(i) is computed as the fixed point of   m[i] <- min(m[i], min_{j ~ i} m[j]),
m[i] = i initially: the minimum over everything reachable from i, i.e. over C(i).
"""
from __future__ import annotations

import numpy as np


def t2_f32(d: float) -> np.float32:
    d = np.float32(d)
    return np.float32(d * d)


def d2_f32(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """fp32 squared distance in the fixed order; a, b broadcastable [..., 3] float32."""
    a = np.asarray(a, dtype=np.float32)
    b = np.asarray(b, dtype=np.float32)
    dx = b[..., 0] - a[..., 0]
    dy = b[..., 1] - a[..., 1]
    dz = b[..., 2] - a[..., 2]
    return (dx * dx + dy * dy) + dz * dz


def pred_f32(a, b, d: float) -> np.ndarray:
    return d2_f32(a, b) <= t2_f32(d)


def edges(points: np.ndarray, d: float, chunk: int = 2048):
    """All unordered pairs (i<j) with pred true, by exhaustive comparison."""
    p = np.ascontiguousarray(points, dtype=np.float32)
    n = p.shape[0]
    I, J = [], []
    for s in range(0, n, chunk):
        blk = p[s:s + chunk]
        m = pred_f32(blk[:, None, :], p[None, :, :], d)     # [chunk, n]
        ii, jj = np.nonzero(m)
        ii = ii + s
        keep = ii < jj
        I.append(ii[keep])
        J.append(jj[keep])
    if not I:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(I), np.concatenate(J)


def brute_labels_unfiltered(points: np.ndarray, d: float) -> np.ndarray:
    """labels[i] = min C(i) (no size filter)."""
    n = np.asarray(points).shape[0]
    m = np.arange(n, dtype=np.int64)
    I, J = edges(points, d)
    while True:
        old = m.copy()
        mi, mj = m[I], m[J]
        np.minimum.at(m, I, mj)
        np.minimum.at(m, J, mi)
        if np.array_equal(m, old):
            return m


def brute_fec(points: np.ndarray, d: float, min_size: int = 1, max_size: int = 2**62) -> np.ndarray:
    m = brute_labels_unfiltered(points, d)
    n = m.shape[0]
    size = np.bincount(m, minlength=n)[m] if n else m
    keep = (size >= min_size) & (size <= max_size)
    return np.where(keep, m, -1).astype(np.int32)
