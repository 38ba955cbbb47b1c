"""Pins for the oracle (CPU, `-m "not gpu"`).

The oracle is pinned to things other than itself:
  * exact rational arithmetic with an independently written IEEE binary32 round-to-nearest
    (the fixed-order, no-FMA predicate of readings A1-A3, Eq. 1);
  * closed forms (3-4-5, axis pairs at exactly d, d + 1 ulp, dyadic lattices);
  * hand-computed worked examples under tests/golden/ (each with its citation);
  * the O(n^2) definition (oracle/brute.py) and a library routine
    (scipy.sparse.csgraph.connected_components) on 200+ random clouds;
  * invariants at C1/C2 size (edge completeness, connectivity of every label class,
    min-index canonical form, size filter, permutation invariance).
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ----------------------------------------------------------------------------------------
# Independent IEEE-754 binary32 round-to-nearest-even on exact rationals.
# ----------------------------------------------------------------------------------------
def rn32(q: Fraction) -> Fraction:
    if q == 0:
        return Fraction(0)
    sign = -1 if q < 0 else 1
    a = abs(q)
    e = a.numerator.bit_length() - a.denominator.bit_length()
    if Fraction(2) ** e > a:
        e -= 1
    while Fraction(2) ** (e + 1) <= a:
        e += 1
    e = max(e, -126)                      # below 2^-126: subnormal quantum 2^-149
    quantum = Fraction(2) ** (e - 23)
    m = a / quantum
    fl = m.numerator // m.denominator
    rem = m - fl
    if rem > Fraction(1, 2) or (rem == Fraction(1, 2) and fl % 2 == 1):
        fl += 1
    return sign * fl * quantum


def exact_d2(a, b, fused=False) -> Fraction:
    """d2 with one binary32 rounding per operation, in the fixed order of reading A2.
    fused=True models an FMA-contracted build: fma(dz,dz, fma(dy,dy, dx*dx))."""
    d = [rn32(Fraction(float(b[k])) - Fraction(float(a[k]))) for k in range(3)]
    if not fused:
        sx, sy, sz = (rn32(v * v) for v in d)
        return rn32(rn32(sx + sy) + sz)
    sx = rn32(d[0] * d[0])
    s = rn32(d[1] * d[1] + sx)
    return rn32(d[2] * d[2] + s)


def test_rn32_selfcheck_against_numpy_casts():
    # the rounding helper agrees with numpy's float64->float32 cast where that is exact
    rng = np.random.default_rng(5)
    for v in rng.normal(size=200) * 10.0 ** rng.integers(-30, 30, size=200):
        assert rn32(Fraction(float(v))) == Fraction(float(np.float32(v)))


# ----------------------------------------------------------------------------------------
# Predicate pins
# ----------------------------------------------------------------------------------------
def test_pred_345_spec_examples():
    assert oracle.pred([0, 0, 0], [3, 4, 0], 5.0)          # SPEC.md L64, boundary inclusive
    assert not oracle.pred([0, 0, 0], [3, 4, 0], 4.999)
    assert oracle.pred([1, 2, 3], [1, 2, 3], 1e-3)         # SPEC.md L63 (identity)


def test_t2_is_single_rounding():
    rng = np.random.default_rng(1)
    for d in rng.uniform(1e-3, 1e3, size=500).astype(np.float32):
        assert Fraction(oracle.t2(float(d))) == rn32(Fraction(float(d)) ** 2)


def test_axis_pair_at_exactly_d_true_and_next_ulp_false():
    rng = np.random.default_rng(2)
    ds = (rng.uniform(0.01, 50.0, size=2000)).astype(np.float32)
    for d in ds:
        base = np.float32(rng.uniform(-100, 100))
        a = np.array([0.0, 0.0, 0.0], np.float32)
        b = np.array([d, 0.0, 0.0], np.float32)
        assert oracle.pred(a, b, float(d))
        nxt = np.nextafter(d, np.float32(np.inf))
        assert not oracle.pred(a, np.array([nxt, 0, 0], np.float32), float(d))
        # translated copies: the difference is no longer exact in general, so compare with
        # the exact-rational model instead of a closed form
        a2 = np.array([base, 0, 0], np.float32)
        b2 = np.array([base + d, 0, 0], np.float32)
        t2 = rn32(Fraction(float(d)) ** 2)
        assert oracle.pred(a2, b2, float(d)) == (exact_d2(a2, b2) <= t2)


def test_d2_matches_exact_rounding_model_and_is_not_fma():
    rng = np.random.default_rng(3)
    n_fma_diff = 0
    for _ in range(3000):
        a = rng.uniform(-50, 50, size=3).astype(np.float32)
        b = (a + rng.normal(0, 1.0, size=3)).astype(np.float32)
        got = Fraction(float(oracle.d2(a, b)))
        assert got == exact_d2(a, b)
        if exact_d2(a, b, fused=True) != got:
            n_fma_diff += 1
    # the pin discriminates: a contracted (FMA) build would differ on many pairs
    assert n_fma_diff > 100


def test_fma_trap_pairs_decided_unfused():
    """Pairs whose fused and unfused d2 straddle t2: the oracle must take the unfused side."""
    rng = np.random.default_rng(4)
    found = 0
    for _ in range(200000):
        d = np.float32(rng.uniform(0.1, 2.0))
        a = rng.uniform(-20, 20, size=3).astype(np.float32)
        v = rng.normal(size=3)
        v = v / np.linalg.norm(v) * float(d) * (1 + rng.normal(0, 2e-7))
        b = (a + v).astype(np.float32)
        t2 = rn32(Fraction(float(d)) ** 2)
        u, f = exact_d2(a, b), exact_d2(a, b, fused=True)
        if (u <= t2) != (f <= t2):
            found += 1
            assert oracle.pred(a, b, float(d)) == (u <= t2)
            if found >= 25:
                break
    assert found >= 5


# ----------------------------------------------------------------------------------------
# Worked examples (tests/golden/spec_examples.json)
# ----------------------------------------------------------------------------------------
def _golden_cases():
    with open(os.path.join(GOLDEN, "spec_examples.json")) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
def test_golden_examples(case):
    pts = np.array(case["points"], dtype=np.float32).reshape(-1, 3)
    want = np.array(case["labels"], dtype=np.int32)
    got = oracle.fec(pts, case["d_th"], case["min_size"], case["max_size"])
    np.testing.assert_array_equal(got, want)
    got_b = oracle.brute_fec(pts, case["d_th"], case["min_size"], case["max_size"])
    np.testing.assert_array_equal(got_b, want)


# ----------------------------------------------------------------------------------------
# Closed-form constructions
# ----------------------------------------------------------------------------------------
def test_chain_at_dyadic_spacing_is_one_component():
    for d in (0.25, 0.5, 0.75, 1.0, 3.0):
        for axis in range(3):
            p = np.zeros((64, 3), np.float32)
            p[:, axis] = np.arange(64) * d
            perm = np.random.default_rng(axis).permutation(64)
            lab = oracle.fec(p[perm], d)
            assert (lab == lab.min()).all() and lab.min() == 0


def test_chain_at_d_plus_ulp_is_singletons():
    for d in (0.25, 0.5, 1.0, 2.0):
        x = [np.float32(0.0)]
        for _ in range(19):   # next point: one ulp beyond x + d
            x.append(np.nextafter(np.float32(x[-1] + np.float32(d)), np.float32(np.inf)))
        p = np.zeros((20, 3), np.float32)
        p[:, 0] = x
        # every fp32 gap exceeds d, so fl(gap^2) > fl(d^2) = t2 (monotone rounding, gap >= d+ulp)
        gaps = np.diff(p[:, 0])
        assert (gaps > np.float32(d)).all()
        lab = oracle.fec(p, d)
        np.testing.assert_array_equal(lab, np.arange(20))


def test_separated_lattices_known_min_indices():
    rng = np.random.default_rng(7)
    blocks, want = [], []
    for k in range(6):
        g = np.stack(np.meshgrid(*[np.arange(4)] * 3, indexing="ij"), -1).reshape(-1, 3)
        blocks.append(g * 0.5 + k * 100.0)
    p = np.concatenate(blocks).astype(np.float32)
    comp = np.repeat(np.arange(6), 64)
    perm = rng.permutation(p.shape[0])
    p, comp = p[perm], comp[perm]
    want = np.array([np.nonzero(comp == c)[0].min() for c in comp])
    np.testing.assert_array_equal(oracle.fec(p, 0.5), want)
    # just below the lattice spacing everything falls apart
    np.testing.assert_array_equal(oracle.fec(p, 0.49), np.arange(p.shape[0]))


def test_all_identical_points():
    p = np.full((1000, 3), 3.25, np.float32)
    np.testing.assert_array_equal(oracle.fec(p, 1e-3), np.zeros(1000, np.int32))
    np.testing.assert_array_equal(oracle.fec(p, 1e-3, 1001, 2000), np.full(1000, -1, np.int32))


def test_error_paths():
    p = np.zeros((3, 3), np.float32)
    for bad_d in (0.0, -1.0, float("nan"), float("inf"), 1e-20, 1e20):
        with pytest.raises(oracle.OracleError) as e:
            oracle.fec(p, bad_d)
        assert e.value.code == oracle.ERR_INVALID_ARGUMENT
    with pytest.raises(oracle.OracleError):
        oracle.fec(p, 1.0, 5, 4)
    q = p.copy()
    q[1, 2] = np.nan
    with pytest.raises(oracle.OracleError) as e:
        oracle.fec(q, 1.0)
    assert e.value.code == oracle.ERR_NONFINITE
    q[1, 2] = np.inf
    with pytest.raises(oracle.OracleError):
        oracle.fec(q, 1.0)
    # smallest / largest valid d (t2 normal and finite): reading A13
    assert oracle.fec(p, float(np.float32(2.0 ** -63)))[0] == 0
    assert oracle.fec(p, float(np.nextafter(np.float32(2.0 ** 64), np.float32(0))))[0] == 0


# ----------------------------------------------------------------------------------------
# Oracle == O(n^2) definition == library routine on random clouds
# ----------------------------------------------------------------------------------------
@pytest.mark.parametrize("chunk", range(4))
def test_oracle_equals_bruteforce_random_clouds(chunk):
    for seed in range(chunk * 55, chunk * 55 + 55):
        p, d, geom = synth.random_cloud(seed)
        rng = np.random.default_rng(seed)
        mn = int(rng.integers(0, 6))
        mx = int(rng.integers(max(mn, 1), 3000))
        got = oracle.fec(p, d, mn, mx)
        want = oracle.brute_fec(p, d, mn, mx)
        assert np.array_equal(got, want), (seed, geom)


def test_bruteforce_equals_scipy_connected_components():
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    from oracle.brute import edges
    for seed in range(40):
        p, d, geom = synth.random_cloud(seed, n=600)
        n = p.shape[0]
        I, J = edges(p, d)
        A = coo_matrix((np.ones(I.shape[0]), (I, J)), shape=(n, n))
        _, comp = connected_components(A, directed=False)
        # canonical form: min index per scipy component
        mins = np.full(comp.max() + 1, n)
        np.minimum.at(mins, comp, np.arange(n))
        np.testing.assert_array_equal(oracle.brute_labels_unfiltered(p, d), mins[comp])
        np.testing.assert_array_equal(oracle.fec(p, d), mins[comp])


# ----------------------------------------------------------------------------------------
# Invariants on BASELINE configs C1 (full) and C2 (full)
# ----------------------------------------------------------------------------------------
def _check_invariants(p, d, mn, mx):
    from oracle.brute import edges
    n = p.shape[0]
    un = oracle.fec(p, d)                       # unfiltered: min C(i)
    idx = np.arange(n)
    assert (un <= idx).all() and (un[un] == un).all()
    I, J = edges(p, d)
    assert (un[I] == un[J]).all()               # every pred-true pair shares a label
    # every label class is connected: min-propagation restricted to the edges reaches it
    m = idx.copy()
    while True:
        old = m.copy()
        np.minimum.at(m, I, m[J])
        np.minimum.at(m, J, old[I])
        if np.array_equal(m, old):
            break
    np.testing.assert_array_equal(m, un)
    lab = oracle.fec(p, d, mn, mx)
    size = np.bincount(un, minlength=n)[un]
    keep = (size >= mn) & (size <= mx)
    np.testing.assert_array_equal(lab, np.where(keep, un, -1))
    return un


def test_invariants_c1():
    w = synth.make_config("C1")
    un = _check_invariants(w.points, w.d_th, w.min_size, w.max_size)
    sizes = np.bincount(un)
    # 20 blobs of 400 points (sigma 0.3 m, d 0.5 m) -> about 20 big clusters
    assert 15 <= (sizes >= 300).sum() <= 25


def test_invariants_c2_scan():
    w = synth.make_config("C2")
    assert 20_000 < w.n < 70_000
    _check_invariants(w.points, w.d_th, w.min_size, w.max_size)


def test_permutation_invariance_of_partition():
    w = synth.make_config("C1")
    a = oracle.fec(w.points, w.d_th)
    perm = np.random.default_rng(9).permutation(w.n)
    b = oracle.fec(w.points[perm], w.d_th)
    # same partition: the pair (a[perm], b) is a bijection between label values
    pairs = np.unique(np.stack([a[perm], b], 1), axis=0)
    assert len(np.unique(pairs[:, 0])) == len(pairs) == len(np.unique(pairs[:, 1]))


def test_component_queries_match_full_run():
    w = synth.make_config("C2")
    full = oracle.fec(w.points, w.d_th)
    size = np.bincount(full, minlength=w.n)
    ix = oracle.Index(w.points, w.d_th)
    for i in np.random.default_rng(0).integers(0, w.n, size=50):
        mn, sz = ix.component(int(i))
        assert mn == full[i] and sz == size[full[i]]
    ix.close()
