"""Pins of the AP oracle (oracle/metrics.py) and of the voxel-fill generator
(synth.voxel_clusters): SPEC's hand-computed examples, the greedy consumption
rule on a hand-built case, label-renaming invariance, and the generator's ground truth being
exactly the connected-component partition at its recommended d_th, so clustering
it reaches AP = 1 (the paper's "precision approximate to 1")."""
import numpy as np
import pytest

import oracle
import synth
from oracle.metrics import average_precision


def test_spec_examples():
    gt = np.array([1] * 10 + [2] * 10)
    assert average_precision(gt - 1, gt)["ap"] == 1.0                       # pred == gt
    r = average_precision(np.zeros(20, int), gt)                            # merged: IoU 0.5
    assert (r["tp"], r["fp"], r["ap"]) == (0, 1, 0.0)
    gt = np.ones(100, int)
    pred = np.array([0] * 75 + [75] * 25)                                   # split 75 / 25
    r = average_precision(pred, gt)
    assert (r["tp"], r["fp"], r["ap"]) == (1, 1, 0.5)


def test_threshold_is_inclusive_and_gt0_excluded():
    gt = np.array([1] * 4 + [0] * 50)
    pred = np.array([0, 0, 0, 7] + [0] * 50)            # the 50 gt-0 points do not count
    r = average_precision(pred, gt)
    assert r["tp"] == 1 and r["fp"] == 1                # IoU 3/4 = 0.75 exactly -> TP; {7} FP
    assert average_precision(pred, gt, 0.76)["tp"] == 0


def test_greedy_consumption():
    """gt 1 = points 0-5, gt 2 = points 6-9.  The larger predicted cluster A = {0,1,6..9} (size 6)
    goes first: IoU(A,1) = 2/10, IoU(A,2) = 4/6 -> it consumes gt 2 as an FP (4/6 < 0.75);
    B = {2..5}: IoU(B,1) = 4/6 -> FP.  Moving points 0,1 into B makes both exact -> AP = 1."""
    gt = np.array([1, 1, 1, 1, 1, 1, 2, 2, 2, 2])
    pred = np.array([5, 5, 9, 9, 9, 9, 5, 5, 5, 5])     # A=5: {0,1,6..9} size 6; B=9: {2..5} size 4
    r = average_precision(pred, gt)
    # A: IoU(A,1) = 2/8, IoU(A,2) = 4/6 -> takes gt 2 (0.667 < 0.75: FP); B: IoU(B,1) = 4/6 -> FP
    assert (r["tp"], r["fp"]) == (0, 2)
    pred2 = np.array([5, 5, 9, 9, 9, 9, 5, 5, 5, 5])
    pred2[[0, 1]] = 9                                   # A = gt 2 exactly, B = gt 1 exactly
    assert average_precision(pred2, gt)["ap"] == 1.0


def test_empty_conventions():
    assert average_precision(np.zeros(0, int), np.zeros(0, int))["ap"] == 1.0
    assert average_precision(np.full(5, -1), np.ones(5, int))["ap"] == 0.0
    assert average_precision(np.arange(5), np.zeros(5, int))["ap"] == 1.0   # nothing counted


@pytest.mark.parametrize("seed", range(5))
def test_label_renaming_invariance(seed):
    """Order-preserving renaming of predicted and gt labels changes nothing (ties are broken
    by label order); AP stays in [0, 1]; n_gt counts the nonzero gt labels."""
    rng = np.random.default_rng(seed)
    n = 500
    gt = rng.integers(0, 12, n)
    pred = np.where(rng.random(n) < 0.8, gt * 3, rng.integers(-1, 40, n))
    r0 = average_precision(pred, gt)
    r1 = average_precision(np.where(pred < 0, -1, 7 * pred + 2), np.where(gt == 0, 0, 5 * gt + 1))
    assert (r0["tp"], r0["fp"], r0["n_pred"], r0["n_gt"]) == (r1["tp"], r1["fp"], r1["n_pred"], r1["n_gt"])
    assert 0.0 <= r0["ap"] <= 1.0 and r0["n_gt"] == len(set(gt[gt != 0].tolist()))


def test_voxel_generator_rejects_unseparated_configs():
    """SPEC.md L357's validity rule (recommended d_th = 1.1 x pitch must stay below the voxel
    edge).  SPEC's own n=2, m=8 example (L365: pitch = voxel edge) violates it: with a stride-2
    lattice the gap between voxels is one edge < 1.1 pitch, so it is rejected (reading M5)."""
    with pytest.raises(ValueError):
        synth.voxel_clusters(2, 8)


@pytest.mark.parametrize("n,m,sigma", [(1, 1, 0.0), (2, 27, 0.0), (100, 200, 0.0), (30, 50, 0.05)])
def test_voxel_generator_ground_truth_is_the_cc_partition(n, m, sigma):
    pts, gt, d = synth.voxel_clusters(n, m, shift_sigma=sigma, seed=n)
    assert pts.shape == (n * m, 3) and sorted(set(gt.tolist())) == list(range(1, n + 1))
    lab = oracle.fec(pts, d)
    if sigma == 0.0:
        # exactly the gt partition (S:L363 invariant) and AP = 1
        first = {}
        for i, g in enumerate(gt.tolist()):
            first.setdefault(g, i)
        assert np.array_equal(lab, np.array([first[g] for g in gt.tolist()]))
        assert average_precision(lab, gt)["ap"] == 1.0
    else:
        # clusters never merge across voxels (clamped shift, stride-2 lattice)
        for k in set(lab.tolist()):
            assert len(set(gt[lab == k].tolist())) == 1
