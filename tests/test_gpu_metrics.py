"""GPU parity of the AP metric (include/fec_metrics.h) against the oracle
(oracle/metrics.py) through the C ABI: TP, FP and the cluster counts equal exactly.  Cases:
SPEC's examples, the greedy-consumption case, random label noise, the clustering path's own
output on the voxel generator (AP = 1) and on LiDAR-like data, empty and all-noise inputs,
out-of-range labels (status -1), ragged sizes across radix tiles."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
from oracle.metrics import average_precision as ap_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2208_07678_b200 as fec
    fec.lib()
    return fec


def check(fec, pred, gt, thr=0.75):
    pred = np.asarray(pred, np.int32)
    gt = np.asarray(gt, np.int32)
    got = fec.average_precision(torch.from_numpy(pred).cuda(), torch.from_numpy(gt).cuda(), thr)
    want = ap_oracle(pred, gt, thr)
    assert got["status"] == 0
    for k in ("tp", "fp", "n_pred", "n_gt"):
        assert got[k] == want[k], (k, got, want)
    assert got["ap"] == want["ap"]
    return got


def test_spec_examples(fec):
    gt = np.array([1] * 10 + [2] * 10)
    assert check(fec, gt - 1, gt)["ap"] == 1.0
    assert check(fec, np.zeros(20), gt)["ap"] == 0.0
    assert check(fec, np.array([0] * 75 + [75] * 25), np.ones(100))["ap"] == 0.5
    check(fec, [5, 5, 9, 9, 9, 9, 5, 5, 5, 5], [1, 1, 1, 1, 1, 1, 2, 2, 2, 2])
    check(fec, [0, 0, 0, 7] + [0] * 50, [1] * 4 + [0] * 50)
    check(fec, [0, 0, 0, 7] + [0] * 50, [1] * 4 + [0] * 50, 0.76)


def test_empty_and_noise(fec):
    check(fec, np.zeros(0), np.zeros(0))
    check(fec, np.full(7, -1), np.ones(7))
    check(fec, np.arange(9), np.zeros(9))


@pytest.mark.parametrize("seed", range(6))
def test_random_label_noise(seed, fec):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 70000))
    k = int(rng.integers(1, 300))
    gt = rng.integers(0, k + 1, n)
    base = rng.permutation(n)[:k + 1]                      # pred labels are point indices
    pred = np.where(rng.random(n) < rng.uniform(0.3, 0.97), base[gt], rng.integers(-1, n, n))
    check(fec, pred, gt, float(rng.choice([0.5, 0.75, 0.9, 1.0])))


def test_voxel_clusters_through_the_clustering_path(fec):
    pts, gt, d = synth.voxel_clusters(300, 200, seed=3)
    lab = fec.cluster(torch.from_numpy(pts).cuda(), d)
    got = fec.average_precision(lab, torch.from_numpy(gt).cuda())
    assert got["ap"] == 1.0 and got["tp"] == 300
    pts, gt, d = synth.voxel_clusters(200, 100, shift_sigma=0.1, seed=4)
    lab = fec.cluster(torch.from_numpy(pts).cuda(), d).cpu().numpy()
    check(fec, lab, gt)


def test_lidar_scan_against_noisy_truth(fec):
    """C2 scan: oracle labels as 'truth' (ids 1..K), the GPU labels at a smaller radius as the
    prediction -> a realistic mix of matches, splits and noise."""
    w = synth.make_config("C2")
    truth = oracle.fec(w.points, w.d_th, 1, 2**62)
    _, gt = np.unique(truth, return_inverse=True)
    pred = fec.cluster(torch.from_numpy(w.points).cuda(), 0.25, 5).cpu().numpy()
    check(fec, pred, gt.astype(np.int32) + 1)


def test_out_of_range_labels(fec):
    got = fec.average_precision(torch.tensor([0, 5], dtype=torch.int32).cuda(),
                                torch.tensor([1, 1], dtype=torch.int32).cuda())
    assert got["status"] == -1 and got["tp"] == -1
    got = fec.average_precision(torch.tensor([0, 1], dtype=torch.int32).cuda(),
                                torch.tensor([1, 3], dtype=torch.int32).cuda())
    assert got["status"] == -1
