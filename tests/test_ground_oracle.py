"""Pins of the ground-removal oracle against what SPEC/the mathematics fix.

The oracle (oracle/ground_oracle.c + oracle/ground.py) is checked against: SPEC.md's three
worked examples (L313-315), exact rational arithmetic for the fused residual (reading G3),
closed-form planes (axis planes, planes of known normal), geometric invariants of the
cross-product normal (reading G2), brute-force fp64 distances away from the threshold,
the tilt and tie rules (G2/G4), and least-squares optimality of the refinement (G7)."""
import math
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import ground

COS30 = math.cos(math.radians(30.0))


def _round_f32(q: Fraction) -> float:
    """Exact round-to-nearest-even of a rational to binary32 (normal range)."""
    if q == 0:
        return 0.0
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    while Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    scale = Fraction(2) ** (e - 23)          # 24-bit significand
    m = a / scale
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * float(fl * scale)


def _exact_residual(plane, p) -> float:
    nx, ny, nz, off = (Fraction(float(v)) for v in np.asarray(plane, np.float32))
    x, y, z = (Fraction(float(v)) for v in np.asarray(p, np.float32))
    r = Fraction(_round_f32(nx * x + off))
    r = Fraction(_round_f32(ny * y + r))
    return _round_f32(nz * z + r)


def test_residual_is_three_single_rounded_fmas():
    """G3: r = fmaf(nz, z, fmaf(ny, y, fmaf(nx, x, off))) -- exact rational reference.  An
    unfused multiply-add or a double-rounded fp64 path differs on some of these inputs."""
    rng = np.random.default_rng(5)
    unfused_differs = 0
    for _ in range(3000):
        pl = rng.normal(size=4).astype(np.float32)
        p = (rng.normal(size=3) * rng.choice([1.0, 30.0, 1e3])).astype(np.float32)
        got = float(ground.residual(pl, p))
        assert got == _exact_residual(pl, p)
        r = np.float32(np.float32(pl[0] * p[0]) + pl[3])
        r = np.float32(np.float32(pl[1] * p[1]) + r)
        r = np.float32(np.float32(pl[2] * p[2]) + r)
        unfused_differs += float(r) != got
    assert unfused_differs > 0  # the test can tell a fused chain from an unfused one


def test_axis_plane_closed_form():
    p = np.array([[0, 0, 5], [1, 0, 5], [0, 1, 5], [3, 4, 5.25]], np.float32)
    ex, ok, pl = ground.plane(p, [0, 1, 2], COS30)
    assert ex and ok and pl.tolist() == [0.0, 0.0, 1.0, -5.0]
    # orientation: reversed winding gives the same (n_z >= 0) plane
    ex, ok, pl2 = ground.plane(p, [0, 2, 1], COS30)
    assert pl2.tolist() == pl.tolist()
    assert float(ground.residual(pl, p[3])) == 0.25


@pytest.mark.parametrize("seed", range(20))
def test_plane_of_known_normal(seed):
    """Three points on the plane n.p + off = 0 (n of known direction) give back n, off."""
    rng = np.random.default_rng(seed)
    n = rng.normal(size=3)
    n[2] = abs(n[2]) + 0.1
    n /= np.linalg.norm(n)
    off = rng.uniform(-5, 5)
    # two orthonormal in-plane directions
    a = np.cross(n, [1.0, 0.0, 0.0])
    a /= np.linalg.norm(a)
    b = np.cross(n, a)
    base = -off * n
    q = np.stack([base + rng.uniform(-10, 10) * a + rng.uniform(-10, 10) * b for _ in range(3)])
    pts = q.astype(np.float32)
    ex, ok, pl = ground.plane(pts, [0, 1, 2], -1.0)
    assert ex and ok
    assert np.allclose(pl[:3], n, atol=2e-5), (pl, n)
    assert abs(pl[3] - off) < 2e-4
    # invariants: unit length, orthogonal to the two edges, n_z >= 0
    u, v = pts[1].astype(np.float64) - pts[0], pts[2].astype(np.float64) - pts[0]
    assert abs(np.linalg.norm(pl[:3].astype(np.float64)) - 1) < 1e-6
    assert abs(float(pl[:3] @ u)) < 1e-5 * np.linalg.norm(u)
    assert abs(float(pl[:3] @ v)) < 1e-5 * np.linalg.norm(v)
    assert pl[2] >= 0


def test_degenerate_hypotheses_are_invalid():
    p = np.array([[0, 0, 0], [1, 1, 1], [2, 2, 2], [0, 1, 0]], np.float32)
    assert not ground.plane(p, [0, 1, 2], COS30)[0]      # collinear
    assert not ground.plane(p, [0, 0, 3], COS30)[0]      # repeated index
    assert not ground.plane(p, [0, 1, 4], COS30)[0]      # out of range
    assert not ground.plane(p, [-1, 1, 3], COS30)[0]
    ex, ok, _ = ground.plane(np.array([[0, 0, 0], [0, 1, 0], [0, 0, 1]], np.float32), [0, 1, 2], COS30)
    assert ex and not ok                                  # vertical wall: tilt 90 deg


def test_spec_example_plane_plus_box():
    """1,000 points on z=0 + 100 in a box at z in [1,3], threshold 0.1,
    max_tilt 30 deg -> exactly the 1,000 z=0 points removed."""
    p = synth.plane_and_box()
    tri = synth.ransac_triplets(p.shape[0], 100, seed=1)
    r = ground.ransac_ground(p, tri, 0.1, COS30, math.ceil(p.shape[0] / 10))
    assert r.best >= 0 and r.n_inliers == 1000
    assert r.ground[:1000].all() and not r.ground[1000:].any()
    assert r.keep_idx.tolist() == list(range(1000, 1100))
    assert np.array_equal(r.keep_points, p[1000:])
    assert np.allclose(r.refined, [0, 0, 1, 0], atol=1e-12)


def test_spec_example_no_dominant_plane():
    """everything strictly above z=1 with no dominant plane -> unchanged."""
    rng = np.random.default_rng(3)
    p = rng.uniform([0, 0, 1.5], [10, 10, 11.5], size=(2000, 3)).astype(np.float32)
    tri = synth.ransac_triplets(2000, 100, seed=3)
    r = ground.ransac_ground(p, tri, 0.05, COS30, 200)
    assert r.best == -1 and r.n_inliers == 0 and not r.ground.any()
    assert r.keep_idx.tolist() == list(range(2000)) and np.isnan(r.plane).all()


def test_spec_example_two_points():
    """a cloud of 2 points -> unchanged, empty model."""
    p = np.array([[0, 0, 0], [1, 0, 0]], np.float32)
    r = ground.ransac_ground(p, synth.ransac_triplets(2, 10), 0.1, COS30, 1)
    assert r.best == -1 and r.keep_idx.tolist() == [0, 1] and not r.valid.any()


def test_tilt_bound_rejects_the_larger_wall():
    """A vertical wall with more points than the floor: the floor is chosen (tilt, G2)."""
    rng = np.random.default_rng(4)
    wall = np.c_[np.full(1500, 3.0), rng.uniform(-10, 10, 1500), rng.uniform(0.5, 10, 1500)]
    floor = np.c_[rng.uniform(-10, 10, 1000), rng.uniform(-10, 10, 1000), np.zeros(1000)]
    p = np.concatenate([wall, floor]).astype(np.float32)
    tri = synth.ransac_triplets(p.shape[0], 200, seed=4)
    r = ground.ransac_ground(p, tri, 0.05, COS30, 100)
    assert r.n_inliers == 1000 and r.ground[1500:].all() and not r.ground[:1500].any()
    # the wall's hypotheses exist but are tilt-invalid, and they count more inliers
    assert r.counts.max() >= 1500


def test_ties_pick_the_lowest_hypothesis():
    p = synth.plane_and_box()
    tri = np.array([[1000, 1001, 1002], [0, 1, 2], [3, 4, 5], [0, 1, 2]], np.int32)
    r = ground.ransac_ground(p, tri, 0.1, COS30, 1)
    assert r.counts[1] == r.counts[2] == r.counts[3] == 1000
    assert r.best == 1


def test_counts_match_fp64_distance_away_from_threshold():
    """Brute force: every point farther than 1e-4 m from the threshold is an inlier iff its
    fp64 point-plane distance is <= threshold, and the counts are the masks' sums."""
    pts, tri, thr, tilt = synth.make_ground_config("G2")
    planes, valid, cnt = ground.counts(pts, tri[:20], thr, math.cos(math.radians(tilt)))
    P = pts.astype(np.float64)
    checked = 0
    for h in range(20):
        exists = ground.plane(pts, tri[h], -2.0)[0]
        if not exists:
            assert cnt[h] == 0
            continue
        m = ground.inlier_mask(pts, planes[h], thr)
        assert int(m.sum()) == int(cnt[h])
        dist = np.abs(P @ planes[h, :3].astype(np.float64) + float(planes[h, 3]))
        far = np.abs(dist - thr) > 1e-4
        assert far.mean() > 0.99
        assert np.array_equal(m[far], (dist <= thr)[far])
        checked += 1
    assert checked >= 15


def test_refinement_is_the_least_squares_plane():
    """G7: the refined normal minimises the sum of squared residuals (small rotations of
    it only increase it) and the plane passes through the inliers' centroid."""
    pts, tri, thr, tilt = synth.make_ground_config("G2")
    r = ground.ransac_ground(pts, tri, thr, math.cos(math.radians(tilt)), pts.shape[0] // 10)
    q = pts[r.ground].astype(np.float64)
    c = q.mean(0)
    n = r.refined[:3]
    assert abs(np.linalg.norm(n) - 1) < 1e-12 and n[2] > 0
    assert abs(n @ c + r.refined[3]) < 1e-9
    f0 = float(((q - c) @ n) ** 2 @ np.ones(len(q)))
    rng = np.random.default_rng(0)
    for _ in range(20):
        m = n + rng.normal(size=3) * 1e-3
        m /= np.linalg.norm(m)
        assert float((((q - c) @ m) ** 2).sum()) >= f0
    # the scene's ground was tilted by 2 degrees: the fit recovers the tilt
    assert abs(math.degrees(math.acos(n[2])) - 2.0) < 0.1


def test_survivors_partition_the_input():
    pts, tri, thr, tilt = synth.make_ground_config("G2")
    r = ground.ransac_ground(pts, tri, thr, math.cos(math.radians(tilt)), pts.shape[0] // 10)
    assert r.best >= 0
    allidx = np.sort(np.concatenate([r.keep_idx, np.nonzero(r.ground)[0]]))
    assert np.array_equal(allidx, np.arange(pts.shape[0]))
    assert np.all(np.diff(r.keep_idx) > 0)
    # every removed point satisfies the plane-distance bound of the chosen plane
    res = np.array([ground.residual(r.plane, pts[i]) for i in np.nonzero(r.ground)[0][:2000]])
    assert np.all(np.abs(res) <= np.float32(thr))
