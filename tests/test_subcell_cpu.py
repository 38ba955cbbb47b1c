"""The fine sub-cell relations of the dense-grid path, checked on the host.

The dense path joins two 4x4x4 sub-cells without any distance test when they are
"certain" and never tests sub-cells beyond "reach".  Both claims are about the fp32
predicate of Eq. 1, so they are pinned here to that predicate itself
(the oracle's numpy fp32 form), evaluated on points sampled in -- and on the corners of --
the two sub-cell boxes, and to the box geometry written out independently in Python.
No GPU is needed: the tables and the bit-parallel flood fill are host code in libfec.so."""
import itertools

import numpy as np
import pytest

from oracle.brute import pred_f32

fec = pytest.importorskip("paper_2208_07678_b200")


@pytest.fixture(scope="module")
def tables():
    fec.lib()
    return fec.subcell_tables()


def slot_offset(s):
    return (s % 3 - 1, (s // 3) % 3 - 1, s // 9 - 1)


def sub_xyz(a):
    return (a & 3, (a >> 2) & 3, a >> 4)


def offset(s, a, b):
    ox, oy, oz = slot_offset(s)
    ax, ay, az = sub_xyz(a)
    bx, by, bz = sub_xyz(b)
    return (4 * ox + bx - ax, 4 * oy + by - ay, 4 * oz + bz - az)


def test_tables_match_box_geometry(tables):
    """certain <=> the farthest points of the two boxes are within d; reach <=> the nearest
    points are closer than one grid cell c (> d): written with the box extents directly."""
    certain, reach = tables
    q = 0.25  # sub-cell edge in units of c; d = c / (1 + 2^-16)
    dd = 1.0 / (1.0 + 2.0 ** -16)
    for s in range(27):
        for a in range(64):
            want_c = want_r = 0
            for b in range(64):
                o = offset(s, a, b)
                far = sum(((abs(v) + 1) * q) ** 2 for v in o) ** 0.5
                near = sum((max(abs(v) - 1, 0) * q) ** 2 for v in o) ** 0.5
                if far <= 0.95 * dd:
                    want_c |= 1 << b
                if near < 1.0:
                    want_r |= 1 << b
            assert int(certain[s][a]) == want_c, (s, a)
            assert int(reach[s][a]) == want_r, (s, a)


def test_certain_and_reach_against_the_fp32_predicate(tables):
    """Points drawn in the boxes (incl. all box corners): certain pairs are pred-true,
    pairs outside reach are pred-false, for several d and grid origins."""
    certain, reach = tables
    rng = np.random.default_rng(5)
    corners = np.array(list(itertools.product([0.0, 1.0], repeat=3)))
    for d in (0.1, 0.25, 0.35, 1.0, 3.7):
        d32 = float(np.float32(d))
        c = d32 * (1.0 + 2.0 ** -16)
        q = c / 4
        lo = rng.uniform(-500, 500, 3)
        for s in rng.choice(27, 8, replace=False):
            for a in rng.choice(64, 6, replace=False):
                for b in range(64):
                    o = np.array(offset(int(s), int(a), b), float)
                    ca = np.array(sub_xyz(int(a)), float)
                    cb = ca + o
                    if abs(o).max() > 6:
                        continue
                    u = np.concatenate([corners, rng.uniform(0, 1, (24, 3))])
                    w = np.concatenate([corners[::-1], rng.uniform(0, 1, (24, 3))])
                    # stay strictly inside the boxes (floor() puts the upper face in the next box)
                    u = np.clip(u, 0, 1 - 1e-9)
                    w = np.clip(w, 0, 1 - 1e-9)
                    pa = (lo + (ca + u) * q).astype(np.float32)
                    pb = (lo + (cb + w) * q).astype(np.float32)
                    # every pairing of the samples
                    A = np.repeat(pa, len(pb), 0)
                    B = np.tile(pb, (len(pa), 1))
                    # fp32 rounding may move a sample out of its box by an ulp; keep exact members
                    fa = np.floor((A.astype(np.float64) - lo) / q)
                    fb = np.floor((B.astype(np.float64) - lo) / q)
                    keep = (fa == ca).all(1) & (fb == cb).all(1)
                    if not keep.any():
                        continue
                    p = pred_f32(A[keep], B[keep], d32)
                    if (int(certain[s][a]) >> b) & 1:
                        assert p.all(), ("certain pair with a pred-false sample", d, s, a, b)
                    if not (int(reach[s][a]) >> b) & 1:
                        assert not p.any(), ("pair beyond reach with a pred-true sample", d, s, a, b)


def test_dilation_equals_in_cell_certain_relation(tables):
    certain, _ = tables
    for a in range(64):
        assert fec.subcell_dilate(1 << a) == int(certain[13][a]) | (1 << a)


def brute_components(occ, certain):
    bits = [b for b in range(64) if (occ >> b) & 1]
    seen, comps = set(), []
    for b in bits:
        if b in seen:
            continue
        comp, stack = 0, [b]
        seen.add(b)
        while stack:
            x = stack.pop()
            comp |= 1 << x
            for y in bits:
                if y not in seen and (int(certain[13][x]) >> y) & 1:
                    seen.add(y)
                    stack.append(y)
        comps.append(comp)
    return comps


def test_components_partition_and_bound(tables):
    certain, _ = tables
    rng = np.random.default_rng(9)
    masks = [0, 1, (1 << 64) - 1, 0x8000000000000001]
    for density in (0.02, 0.05, 0.1, 0.2, 0.4):
        masks += [int(sum(1 << b for b in range(64) if rng.random() < density)) for _ in range(300)]
    for occ in masks:
        got = fec.subcell_components(occ)
        want = brute_components(occ, certain)
        assert got is not None and len(got) <= 8
        assert sorted(got) == sorted(want), hex(occ)
    # the largest set of pairwise non-certain sub-cells has 8 elements (the bound the
    # dense path's 8 component nodes per cell rely on)
    eight = [(0, 0, 0), (3, 0, 0), (0, 3, 0), (3, 3, 0), (1, 1, 2), (3, 0, 3), (0, 3, 3), (3, 3, 3)]
    occ = sum(1 << (x + 4 * y + 16 * z) for x, y, z in eight)
    assert len(fec.subcell_components(occ)) == 8
