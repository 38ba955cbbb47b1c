"""GPU parity of the batched many-cloud API (fec_cluster_batch_ws, the
paper's per-scan mode): every cloud's labels equal the oracle run on that
cloud alone, bit for bit — including clouds that overlap in space (no edge may join two
clouds), empty and one-point clouds, and the one-cloud-at-a-time fallback."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth

pytestmark = pytest.mark.gpu
HUGE = 2**62


@pytest.fixture(scope="module")
def fec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2208_07678_b200 as fec
    fec.lib()
    return fec


def check_batch(fec, clouds, d, mn=1, mx=HUGE):
    offs = np.concatenate([[0], np.cumsum([len(c) for c in clouds])]).astype(np.int64)
    pts = np.concatenate([np.asarray(c, np.float32).reshape(-1, 3) for c in clouds]) if offs[-1] else \
        np.zeros((0, 3), np.float32)
    got = fec.cluster_batch(torch.from_numpy(pts).cuda(), offs, d, mn, mx).cpu().numpy()
    for k, c in enumerate(clouds):
        want = oracle.fec(np.asarray(c, np.float32).reshape(-1, 3), d, mn, mx)
        g = got[offs[k]:offs[k + 1]]
        if not np.array_equal(g, want):
            bad = np.nonzero(g != want)[0]
            raise AssertionError(f"cloud {k}: {bad.size}/{want.size} differ; first {bad[:5]} got {g[bad[:5]]} "
                                 f"want {want[bad[:5]]}")


@pytest.mark.parametrize("mode", [0, 2, 3, 1], ids=["auto", "keysort", "countsort", "percloud"])
def test_batch_random_overlapping_clouds(fec, mode):
    fec.set_grid_mode(mode)
    try:
        rng = np.random.default_rng(21)
        for trial in range(6):
            nclouds = int(rng.integers(1, 40))
            clouds = []
            for c in range(nclouds):
                n = int(rng.choice([0, 1, 2, 50, 300, 2000]))
                # all clouds in the same region: without the cloud separation they would merge
                p = rng.normal(0, 1.0, (n, 3)) if c % 2 else rng.uniform(-2, 2, (n, 3))
                clouds.append(p.astype(np.float32))
            d = float(rng.uniform(0.05, 0.4))
            check_batch(fec, clouds, d)
            check_batch(fec, clouds, d, 5, 400)
    finally:
        fec.set_grid_mode(0)


def test_batch_of_lidar_scans(fec):
    # 12 single scans (C2 recipe, different seeds/objects) = the paper's per-scan mode
    scans = [synth.lidar_scan(seed=100 + k) for k in range(12)]
    check_batch(fec, scans, 0.35, 50, 25000)


def test_batch_edge_cases(fec):
    check_batch(fec, [np.zeros((0, 3))], 0.5)
    check_batch(fec, [np.zeros((0, 3)), np.array([[1, 2, 3]])], 0.5)
    same = np.array([[0, 0, 0], [0.1, 0, 0]], np.float32)
    check_batch(fec, [same, same, same], 0.5)           # identical clouds stay separate
    far = np.array([[0, 0, 0], [1e4, 1e4, 1e4]], np.float32)
    check_batch(fec, [far, same], 0.5)                  # huge bbox: falls back per cloud
    # argument errors: bad offsets
    t = torch.zeros((4, 3), dtype=torch.float32, device="cuda")
    with pytest.raises(ValueError):
        fec.cluster_batch(t, [0, 2], 0.5)                  # offsets do not end at n
    assert fec.lib().fec_cluster_batch_ws(None, None, 0, 0.5, 1, 10, None, None, 0, None) == -1
