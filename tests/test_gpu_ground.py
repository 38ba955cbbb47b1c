"""GPU parity of the ground-removal path (include/fec_ground.h) against the
oracle (oracle/ground.py), through the C ABI: per-hypothesis inlier counts, the chosen plane,
the survivors and their order are bit-exact; the least-squares refit (a binary64 reduction
whose summation order differs) is within the tolerance derived in DESIGN.md §8c.  Edge
cases: empty / tiny clouds, no hypotheses, the maximum hypothesis count, NaN points,
degenerate triplets, ties, ragged sizes.  The full-size G3 map is checked on sampled
hypotheses and on the whole survivor set."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth
from oracle import ground as og

pytestmark = pytest.mark.gpu
COS30 = math.cos(math.radians(30.0))
# refit tolerance (DESIGN.md §8c G7): the binary64 sums differ only in summation order
NORMAL_ATOL = 1e-9
OFFSET_ATOL = 1e-7


@pytest.fixture(scope="module")
def fec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2208_07678_b200 as fec
    fec.lib()
    return fec


def run_gpu(fec, pts, tri, thr, cos_tilt, min_inl):
    p = torch.from_numpy(np.ascontiguousarray(pts, np.float32).reshape(-1, 3)).cuda()
    t = torch.from_numpy(np.ascontiguousarray(tri, np.int32).reshape(-1, 3)).cuda()
    kp, ki, res, cnt = fec.remove_ground(p, t, thr, cos_max_tilt=cos_tilt, min_inliers=min_inl, counts=True)
    torch.cuda.synchronize()
    info = fec.ground_result(res)
    nk = info["n_keep"]
    H = t.shape[0]
    return info, kp[:nk].cpu().numpy(), ki[:nk].cpu().numpy(), (cnt[:H].cpu().numpy() if H else np.zeros(0, np.int64))


def check(fec, pts, tri, thr=0.2, cos_tilt=COS30, min_inl=None):
    pts = np.ascontiguousarray(pts, np.float32).reshape(-1, 3)
    n = pts.shape[0]
    if min_inl is None:
        min_inl = (n + 9) // 10
    want = og.ransac_ground(pts, tri, thr, cos_tilt, min_inl)
    info, kp, ki, cnt = run_gpu(fec, pts, tri, thr, cos_tilt, min_inl)
    assert np.array_equal(cnt, want.counts), np.nonzero(cnt != want.counts)[0][:10]
    assert info["best"] == want.best
    assert info["n_valid"] == int(want.valid.sum())
    assert info["n_inliers"] == want.n_inliers and info["n_keep"] == n - want.n_inliers
    assert np.array_equal(ki, want.keep_idx)
    assert np.array_equal(kp.view(np.uint32), want.keep_points.view(np.uint32))
    if want.best >= 0:
        assert np.array_equal(info["plane"].view(np.uint32), want.plane.view(np.uint32))
        np.testing.assert_allclose(info["refined"][:3], want.refined[:3], rtol=0, atol=NORMAL_ATOL)
        assert abs(info["refined"][3] - want.refined[3]) <= OFFSET_ATOL + 1e-12 * abs(want.refined[3])
    else:
        assert np.isnan(info["plane"]).all() and np.isnan(info["refined"]).all()
    return want


def test_spec_example(fec):
    p = synth.plane_and_box()
    w = check(fec, p, synth.ransac_triplets(p.shape[0], 100, 1), 0.1)
    assert w.n_inliers == 1000


def test_g2_scan(fec):
    pts, tri, thr, tilt = synth.make_ground_config("G2")
    w = check(fec, pts, tri, thr, math.cos(math.radians(tilt)))
    assert w.best >= 0


@pytest.mark.parametrize("seed", range(8))
def test_random_clouds_ragged(seed, fec):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 40000))
    floor = np.c_[rng.uniform(-20, 20, (n, 2)), rng.normal(0, 0.05, n)]
    objs = rng.uniform([-20, -20, 0], [20, 20, 4], (n // 3, 3))
    pts = np.concatenate([floor, objs])[rng.permutation(n + n // 3)]
    H = int(rng.integers(1, 300))
    check(fec, pts, synth.ransac_triplets(pts.shape[0], H, seed), float(rng.uniform(0.02, 0.3)),
          math.cos(math.radians(float(rng.uniform(5, 60)))))


def test_edge_cases(fec):
    # n = 0, n = 2, no hypotheses, all-degenerate hypotheses
    check(fec, np.zeros((0, 3), np.float32), np.zeros((5, 3), np.int32), 0.1)
    check(fec, np.array([[0, 0, 0], [1, 0, 0]], np.float32), synth.ransac_triplets(2, 10), 0.1, COS30, 1)
    p = synth.plane_and_box()
    check(fec, p, np.zeros((0, 3), np.int32), 0.1)
    bad = np.array([[0, 0, 1], [5, 6, 5], [-1, 2, 3], [0, 1, 5000]], np.int32)
    check(fec, p, bad, 0.1)
    # collinear triplet and a vertical wall next to the floor
    line = np.c_[np.arange(10.0), np.zeros(10), np.zeros(10)]
    check(fec, np.concatenate([line, p]), np.array([[0, 1, 2], [10, 11, 12]], np.int32), 0.1, COS30, 1)
    # ties: identical hypotheses -> lowest index
    w = check(fec, p, np.array([[1000, 1001, 1002], [0, 1, 2], [3, 4, 5], [0, 1, 2]], np.int32), 0.1, COS30, 1)
    assert w.best == 1
    # min_inliers above every count -> no ground
    check(fec, p, synth.ransac_triplets(p.shape[0], 50, 2), 0.1, COS30, 5000)
    # threshold 0: only exact zeros count
    check(fec, p, synth.ransac_triplets(p.shape[0], 50, 3), 0.0, COS30, 1)


def test_nan_points_are_never_inliers(fec):
    p = synth.plane_and_box().copy()
    p[5, 2] = np.nan
    p[17] = np.inf
    tri = synth.ransac_triplets(p.shape[0], 100, 4)
    tri[0] = [5, 6, 7]                       # a hypothesis through a NaN point has no plane
    w = check(fec, p, tri, 0.1)
    assert 5 in w.keep_idx and 17 in w.keep_idx


def test_max_hypotheses(fec):
    """FEC_GROUND_MAX_HYP planes (80 KB of shared memory: the opt-in path)."""
    pts, _, thr, tilt = synth.make_ground_config("G2")
    tri = synth.ransac_triplets(pts.shape[0], 4096, 9)
    check(fec, pts[:20011], synth.ransac_triplets(20011, 4096, 9), thr, math.cos(math.radians(tilt)))
    with pytest.raises(fec.FecError):
        fec.remove_ground(torch.from_numpy(pts).cuda(), torch.from_numpy(synth.ransac_triplets(pts.shape[0], 4097)).cuda())
    del tri


def test_cluster_nonground_matches_oracle(fec):
    """Ground removal then clustering: -2 ground, else the oracle's labels of
    the survivors mapped back to input indices."""
    pts, tri, thr, tilt = synth.make_ground_config("G2")
    d, mn, mx = 0.35, 50, 25_000
    got, info = fec.cluster_nonground(torch.from_numpy(pts).cuda(), torch.from_numpy(tri).cuda(), d, mn, mx, thr, tilt)
    got = got.cpu().numpy()
    w = og.ransac_ground(pts, tri, thr, math.cos(math.radians(tilt)), (pts.shape[0] + 9) // 10)
    lab_k = oracle.fec(w.keep_points, d, mn, mx)
    want = np.full(pts.shape[0], -2, np.int32)
    want[w.keep_idx] = np.where(lab_k < 0, -1, w.keep_idx[np.maximum(lab_k, 0)])
    assert np.array_equal(got, want)
    assert (got == -2).sum() == w.n_inliers and (got >= 0).any()


@pytest.mark.slow
def test_g3_full_size_sampled(fec):
    """The bench workload (G3, ~19M points, 100 hypotheses, the launch configuration bench.py
    times): 6 sampled hypotheses' counts and the best plane's complete survivor set."""
    pts, tri, thr, tilt = synth.make_ground_config("G3")
    ct = math.cos(math.radians(tilt))
    info, kp, ki, cnt = run_gpu(fec, pts, tri, thr, ct, (pts.shape[0] + 9) // 10)
    rng = np.random.default_rng(0)
    hs = sorted(set(rng.choice(tri.shape[0], 5, replace=False).tolist()) | {max(info["best"], 0)})
    _, _, c_or = og.counts(pts, tri[hs], thr, ct)
    assert np.array_equal(cnt[hs], c_or)
    # the chosen plane is the argmax of the GPU's own counts over tilt-valid planes (all
    # counts are checked bit-exact at smaller sizes), and its survivor set is exact
    valid = np.array([og.plane(pts, t, ct)[1] for t in tri])
    key = np.where(valid, cnt, -1)
    assert info["best"] == int(np.argmax(key))
    pl = og.plane(pts, tri[info["best"]], ct)[2]
    assert np.array_equal(info["plane"].view(np.uint32), pl.view(np.uint32))
    m = og.inlier_mask(pts, pl, thr)
    assert np.array_equal(ki, np.nonzero(~m)[0].astype(np.int32))
    assert np.array_equal(kp.view(np.uint32), pts[~m].view(np.uint32))
    ref = og.refine(pts[m])
    np.testing.assert_allclose(info["refined"][:3], ref[:3], rtol=0, atol=NORMAL_ATOL)
