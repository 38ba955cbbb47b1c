"""The literal Algorithm 1 comparator (oracle/literal.py) against SPEC's worked
examples and the CC oracle: on every input its partition refines the exact
connected components, equals them on SPEC's examples (including the bridge-last chain, which
exercises the segment merge loop), and differs on SURVEY finding 1's counterexample."""
import numpy as np
import pytest

import oracle
import synth
from oracle.literal import canonical, literal_fec, refines


def test_spec_examples():
    r = literal_fec(np.array([[0, 0, 0], [0.5, 0, 0]]), 1.0)
    assert r.labels.tolist() == [1, 1]
    r = literal_fec(np.array([[0, 0, 0], [10, 0, 0]]), 1.0)
    assert r.labels.tolist() == [1, 2]
    # bridge point LAST: points 0 and 1 get provisional segments 1 and 2, point 2 merges them
    r = literal_fec(np.array([[0, 0, 0], [1.8, 0, 0], [0.9, 0, 0]]), 1.0)
    assert len(set(r.labels.tolist())) == 1
    assert r.neighbor_queries == 2 and r.merge_relabels == 0
    # two well-separated blobs, shuffled: the oracle's 2 components
    rng = np.random.default_rng(0)
    pts = np.concatenate([rng.normal(0, 0.3, (250, 3)), rng.normal(20, 0.3, (250, 3))])[rng.permutation(500)]
    pts = pts.astype(np.float32)
    r = literal_fec(pts, 2.0)
    assert np.array_equal(canonical(r.labels), oracle.brute_fec(pts, 2.0))


def test_merge_loop_fires():
    """Segments 1 = {0, 3} and 2 = {1, 4} exist before the query of the unlabelled bridge 2,
    whose neighbourhood holds both: the segment merge loop sweeps segment 2 into 1."""
    pts = np.array([[0, 0, 0], [3, 0, 0], [1.5, 0, 0], [0.8, 0, 0], [2.2, 0, 0]], np.float32)
    r = literal_fec(pts, 1.0)
    assert r.labels.tolist() == [1, 1, 1, 1, 1]
    assert r.neighbor_queries == 3 and r.merge_relabels == 1 and r.points_relabelled == 2


def test_finding_1_counterexample():
    """x = 0, 2.25, 0.75, 1.5 with d = 1 (SURVEY finding 1): literal FEC gives {0,2} and {1,3};
    the exact CC is one component (0-0.75-1.5-2.25, each gap 0.75)."""
    pts = np.array([[0, 0, 0], [2.25, 0, 0], [0.75, 0, 0], [1.5, 0, 0]], np.float32)
    r = literal_fec(pts, 1.0)
    assert canonical(r.labels).tolist() == [0, 1, 0, 1]
    assert oracle.brute_fec(pts, 1.0).tolist() == [0, 0, 0, 0]
    assert refines(canonical(r.labels), oracle.brute_fec(pts, 1.0))


@pytest.mark.parametrize("seed", range(30))
def test_literal_partition_refines_exact_cc(seed):
    pts, d, _ = synth.random_cloud(seed, n=int(np.random.default_rng(seed).integers(1, 400)))
    want = oracle.fec(pts, d)
    r = literal_fec(pts, d)
    got = canonical(r.labels)
    assert refines(got, want)
    # counters: every segment label ever created came from one query
    assert len(set(r.labels.tolist())) <= r.neighbor_queries <= len(pts)
    # th_max caps the neighbourhood: still a refinement of the exact CC
    rc = literal_fec(pts, d, th_max=3)
    assert refines(canonical(rc.labels), want)


def test_refinement_gap_is_common_on_uniform_clouds():
    """How often the literal procedure differs from exact CC (documented in DESIGN.md §8d)."""
    differ = 0
    for seed in range(40):
        rng = np.random.default_rng(500 + seed)
        pts = rng.uniform(0, 6, (300, 3)).astype(np.float32)
        want = oracle.fec(pts, 0.6)
        got = canonical(literal_fec(pts, 0.6).labels)
        assert refines(got, want)
        differ += not np.array_equal(got, want)
    assert differ > 0
