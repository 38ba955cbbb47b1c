"""AP metric oracle — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Eq. 2 of the paper, AP = TP / (TP + FP), with 0.75 as the point-wise threshold for a true
positive, made concrete by SPEC.md L392-408 (op average_precision) and the
readings M1-M4 of DESIGN.md §8e:

  M1  points whose gt label is 0 are excluded from every count; predicted label -1 (noise)
      is not a predicted cluster (its points still count in |G|);
  M2  predicted clusters in order of descending size |P| (points with gt != 0), ties by
      ascending label;
  M3  each is matched to the still-unmatched gt cluster of largest IoU = |P n G| / |P u G|
      among those it overlaps (ties: smallest gt label), which is then consumed; it is a TP
      iff that IoU >= threshold (compared as  |P n G| >= threshold * |P u G|  in binary64),
      otherwise an FP; a predicted cluster overlapping no unmatched gt cluster is an FP;
  M4  AP = TP/(TP+FP); 1 when there are neither predicted nor gt clusters, 0 when there are
      gt clusters but no predicted ones.
"""
from __future__ import annotations

from collections import Counter, defaultdict

import numpy as np


def average_precision(pred, gt, threshold: float = 0.75) -> dict:
    pred = np.asarray(pred, dtype=np.int64)
    gt = np.asarray(gt, dtype=np.int64)
    if pred.shape != gt.shape:
        raise ValueError("pred and gt must cover the same cloud")
    keep = gt != 0                                              # M1
    P, G = pred[keep], gt[keep]
    size_g = Counter(G.tolist())
    size_p = Counter(P[P >= 0].tolist())
    inter = defaultdict(dict)
    for a, b in zip(P.tolist(), G.tolist()):
        if a >= 0:
            inter[a][b] = inter[a].get(b, 0) + 1
    order = sorted(size_p, key=lambda a: (-size_p[a], a))      # M2
    matched = set()
    tp = fp = 0
    for a in order:                                             # M3
        best, best_c, best_u = None, 0, 1
        for b in sorted(inter[a]):
            if b in matched:
                continue
            c = inter[a][b]
            u = size_p[a] + size_g[b] - c
            if best is None or c * best_u > best_c * u:         # larger IoU; ties keep smaller b
                best, best_c, best_u = b, c, u
        if best is None:
            fp += 1
            continue
        matched.add(best)
        if float(best_c) >= float(threshold) * float(best_u):
            tp += 1
        else:
            fp += 1
    n_gt = len(size_g)
    if tp + fp == 0:
        ap = 1.0 if n_gt == 0 else 0.0                          # M4
    else:
        ap = tp / (tp + fp)
    return {"tp": tp, "fp": fp, "n_pred": len(size_p), "n_gt": n_gt, "ap": ap}
