"""Literal Algorithm 1 comparator — TEST INFRASTRUCTURE ONLY.

The paper's own point-wise procedure, PAPER.md L128-176 (Algorithm 1 "Proposed FEC"), run as
written, with SPEC's resolution of its two pseudocode gaps:

  P.lab <- 0;  segLab <- 1
  for p_i in index order:
    if p_i.lab == 0:
      P_NN <- FindNeighbor(p_i, d_th)   (p_i and its pred-true neighbours; with a cap, p_i
                                         plus the Th_max - 1 nearest others, ties by index --
                                         the kd-tree's max_nn, DESIGN.md §8d reading L1)
      minSegLab <- min(Nonzero(P_NN.lab) U {segLab})
      every p_j in P_NN with label 0 <- minSegLab     (SPEC's fix: the pseudocode never
                                                       assigns a label)
      for every label L > minSegLab among P_NN: sweep the whole cloud, L -> minSegLab
                                                      (segment merge loop)
      segLab++                                                      

FindNeighbor uses the same fp32 predicate as the oracle (Eq. 1, readings A1-A3).  This is NOT
the oracle of the CUDA path: read literally, Algorithm 1 only queries points that are still
unlabelled, so an edge between two already-labelled points of different segments is never
examined and its partition REFINES the exact connected components (SURVEY finding 1).  It
exists to document that gap (tests/test_literal_fec.py) and the paper's counters.
Plain Python + numpy, O(n^2); meant for n <= a few thousand.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .brute import d2_f32, t2_f32


@dataclass
class LiteralResult:
    labels: np.ndarray          # int64 [n], segment labels (>= 1, with gaps)
    neighbor_queries: int       # FindNeighbor calls (points unlabelled when visited)
    merge_relabels: int         # segment-merge sweeps (distinct neighbour labels > minSegLab)
    points_relabelled: int      # points rewritten by the sweeps


def literal_fec(points, d_th: float, th_max: int | None = None) -> LiteralResult:
    p = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
    n = p.shape[0]
    t2 = t2_f32(d_th)
    lab = np.zeros(n, dtype=np.int64)
    seg = 1
    queries = merges = moved = 0
    for i in range(n):
        if lab[i] != 0:
            continue
        queries += 1
        d2 = d2_f32(p[i][None, :], p)
        nn = np.nonzero(d2 <= t2)[0]                     # includes i (d2 = 0)
        if th_max is not None and nn.size > th_max:
            # p_i itself, then the nearest others (ties by index): Th_max points in all
            others = nn[nn != i]
            order = np.lexsort((others, d2[others]))
            nn = np.concatenate([[i], others[order[:max(th_max, 1) - 1]]])
        nz = lab[nn][lab[nn] != 0]
        min_seg = int(min(nz.min(), seg)) if nz.size else seg
        for L in sorted(set(int(v) for v in nz if v > min_seg)):   # segment merge loop
            m = lab == L
            moved += int(m.sum())
            lab[m] = min_seg
            merges += 1
        z = nn[lab[nn] == 0]
        lab[z] = min_seg
        seg += 1
    return LiteralResult(lab, queries, merges, moved)


def canonical(labels) -> np.ndarray:
    """Segment labels -> minimum index of each segment (the oracle's canonical form)."""
    lab = np.asarray(labels)
    out = np.empty(lab.shape[0], dtype=np.int64)
    first = {}
    for i, v in enumerate(lab.tolist()):
        if v not in first:
            first[v] = i
        out[i] = first[v]
    return out


def refines(fine, coarse) -> bool:
    """True iff every class of `fine` lies inside one class of `coarse` (canonical forms)."""
    f = np.asarray(fine)
    c = np.asarray(coarse)
    rep = {}
    for a, b in zip(f.tolist(), c.tolist()):
        if rep.setdefault(a, b) != b:
            return False
    return True
