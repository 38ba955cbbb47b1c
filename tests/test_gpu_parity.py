"""GPU parity: the CUDA path (through the C ABI) vs the oracle, element by element.

Bar: labels are int32 index work, so bit-exact equality.  The oracle runs
live on the same seeded inputs; no expected value comes from the CUDA path."""
import json
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def fec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2208_07678_b200 as fec
    fec.lib()
    return fec


def run_gpu(fec, pts, d, mn=1, mx=2**62):
    t = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float32).reshape(-1, 3)).cuda()
    lab = fec.cluster(t, d, mn, mx)
    torch.cuda.synchronize()
    return lab.cpu().numpy()


def assert_same(got, want, ctx=""):
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{ctx}: {bad.size}/{want.size} labels differ; first {bad[:5]} "
                             f"got {got[bad[:5]]} want {want[bad[:5]]}")


def test_golden_examples_gpu(fec):
    cases = json.load(open(os.path.join(GOLDEN, "spec_examples.json")))["cases"]
    for c in cases:
        pts = np.array(c["points"], dtype=np.float32).reshape(-1, 3)
        got = run_gpu(fec, pts, c["d_th"], c["min_size"], c["max_size"])
        assert_same(got, np.array(c["labels"], np.int32), c["name"])


@pytest.fixture(params=[0, 1, 2, 3], ids=["auto", "hashed", "keysort", "countsort"])
def mode(fec, request):
    fec.set_grid_mode(request.param)
    yield request.param
    fec.set_grid_mode(0)


@pytest.mark.parametrize("chunk", range(4))
def test_random_clouds_bit_exact(fec, mode, chunk):
    for seed in range(chunk * 55, chunk * 55 + 55):
        p, d, geom = synth.random_cloud(seed)
        rng = np.random.default_rng(seed)
        mn = int(rng.integers(0, 6))
        mx = int(rng.integers(max(mn, 1), 3000))
        assert_same(run_gpu(fec, p, d, mn, mx), oracle.fec(p, d, mn, mx), f"seed {seed} {geom} mode {mode}")


def test_larger_random_clouds_span_many_tiles(fec, mode):
    # several radix tiles (4096 keys) and scan tiles, with ragged tails
    for seed, n in ((7, 4097), (8, 20_001), (9, 150_003)):
        p, d, geom = synth.random_cloud(seed, n=n, geometry="blobs")
        assert_same(run_gpu(fec, p, d, 3, 10**6), oracle.fec(p, d, 3, 10**6), f"n={n}")
        p, d, geom = synth.random_cloud(seed, n=n, geometry="uniform")
        assert_same(run_gpu(fec, p, d), oracle.fec(p, d), f"uniform n={n}")


def test_device_predicate_matches_oracle_on_boundary_pairs(fec):
    rng = np.random.default_rng(11)
    m = 200_000
    d = np.float32(0.37)
    a = rng.uniform(-30, 30, size=(m, 3)).astype(np.float32)
    v = rng.normal(size=(m, 3))
    v = v / np.linalg.norm(v, axis=1, keepdims=True) * float(d) * (1 + rng.normal(0, 3e-7, size=(m, 1)))
    b = (a + v).astype(np.float32)
    ok, d2 = fec.debug_pred(torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda(), float(d))
    want_d2 = oracle.d2_f32(a, b)
    np.testing.assert_array_equal(d2.cpu().numpy(), want_d2)          # bit-exact fp32
    np.testing.assert_array_equal(ok.cpu().numpy(), want_d2 <= oracle.brute.t2_f32(d))
    # the set straddles the boundary (both outcomes present)
    o = ok.cpu().numpy()
    assert o.any() and (~o).any()


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_config_full_size(fec, name):
    w = synth.make_config(name)
    assert_same(run_gpu(fec, w.points, w.d_th, w.min_size, w.max_size),
                oracle.fec(w.points, w.d_th, w.min_size, w.max_size), name)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
def test_full_size_label_digest(fec, name):
    """Every config at FULL size (C5: 110M points, the stress config) bit-exact against the
    oracle through stored digests: tests/golden/full_size.json holds the sha256 of each
    config's fp32 input and of the ORACLE's int32 labels, written by
    tools/make_full_size_digests.py, which calls only synth/ and oracle/ (C5's oracle run takes
    ~8 minutes, so it is stored rather than recomputed here).  The input digest is asserted
    first, so a generator that differs on this box fails loudly instead of comparing
    different clouds."""
    import hashlib
    ref = json.load(open(os.path.join(GOLDEN, "full_size.json")))["configs"][name]
    w = synth.make_config(name)
    assert w.n == ref["n"] and synth.sha256_f32(w.points) == ref["input_sha256"], f"{name}: input differs"
    assert (np.float32(w.d_th), w.min_size, w.max_size) == (np.float32(ref["d_th"]), ref["min_size"], ref["max_size"])
    lab = np.ascontiguousarray(run_gpu(fec, w.points, w.d_th, w.min_size, w.max_size), dtype="<i4")
    assert hashlib.sha256(lab.tobytes()).hexdigest() == ref["labels_sha256"], (
        f"{name}: labels differ from the oracle's (noise {(lab < 0).sum()} vs {ref['noise']})")


@pytest.mark.parametrize("name,gmode", [("C3", 1), ("C3", 2), ("C3", 3), ("C4", 1), ("C4", 2), ("C4", 3)])
def test_full_size_label_digest_forced_grid_modes(fec, name, gmode):
    """The paths the automatic plan does not take at full size -- hashed cell index (1), key
    sort (2), counting sort (3) forced on the 9M / 27M-point configs -- against the same stored
    oracle digests (the scaled configs reach these paths too, but with 50x fewer cells, tiles
    and radix buckets)."""
    import hashlib
    ref = json.load(open(os.path.join(GOLDEN, "full_size.json")))["configs"][name]
    w = synth.make_config(name)
    assert synth.sha256_f32(w.points) == ref["input_sha256"], f"{name}: input differs"
    fec.set_grid_mode(gmode)
    try:
        lab = np.ascontiguousarray(run_gpu(fec, w.points, w.d_th, w.min_size, w.max_size), dtype="<i4")
    finally:
        fec.set_grid_mode(0)
    assert hashlib.sha256(lab.tobytes()).hexdigest() == ref["labels_sha256"], (
        f"{name} mode {gmode}: labels differ from the oracle's (noise {(lab < 0).sum()} vs {ref['noise']})")


@pytest.mark.parametrize("name,scale", [("C3", 0.05), ("C4", 0.02), ("C5", 0.02)])
def test_config_scaled(fec, mode, name, scale):
    w = synth.make_config(name, scale=scale)
    assert_same(run_gpu(fec, w.points, w.d_th, w.min_size, w.max_size),
                oracle.fec(w.points, w.d_th, w.min_size, w.max_size), f"{name}@{scale}")
    # and unfiltered
    assert_same(run_gpu(fec, w.points, w.d_th), oracle.fec(w.points, w.d_th), f"{name}@{scale} unfiltered")


def test_host_api_equals_device_api(fec):
    w = synth.make_config("C2")
    dev = run_gpu(fec, w.points, w.d_th, w.min_size, w.max_size)
    host = fec.cluster_host(w.points, w.d_th, w.min_size, w.max_size)
    assert_same(host, dev, "host vs device")
    pinned = torch.from_numpy(w.points).pin_memory()
    host2 = fec.cluster_host(pinned, w.d_th, w.min_size, w.max_size)
    assert_same(host2, dev, "pinned host vs device")


def test_async_host_api_pipelined_over_two_streams(fec):
    """fec_cluster_host_async: six different clouds in flight over two streams (each with its
    own workspace and pinned buffers); every cloud's labels equal the oracle's."""
    clouds = [synth.make_config("C2").points] + [synth.random_cloud(s, n=30_000 + 777 * s)[0] for s in range(5)]
    ds = [0.35] + [float(synth.random_cloud(s, n=10)[1]) for s in range(5)]
    sts = [torch.cuda.Stream() for _ in range(2)]
    nmax = max(len(c) for c in clouds)
    ws = [torch.empty(fec.workspace_bytes_host(nmax), dtype=torch.uint8, device="cuda") for _ in range(2)]
    pins = [torch.from_numpy(c).pin_memory() for c in clouds]
    outs = [torch.empty(len(c), dtype=torch.int32).pin_memory() for c in clouds]
    for k, c in enumerate(clouds):
        fec.cluster_host(pins[k], ds[k], 2, 10**6, out=outs[k], workspace=ws[k % 2], stream=sts[k % 2], sync=False)
    torch.cuda.synchronize()
    for k, c in enumerate(clouds):
        assert_same(outs[k].numpy(), oracle.fec(c, ds[k], 2, 10**6), f"async cloud {k}")


@pytest.mark.parametrize("name,scale", [("C4", 0.02), ("C3", 0.05), ("C5", 0.01)])
def test_shuffled_input_key_path(fec, name, scale):
    """Shuffled input above 2^17 points takes the key-sort path (the a1 coherence test):
    node-tail clouds (shuffled C4 / C3: labels written in input order by k_relabel_in through
    the cell codes of the key path) and a sparse-dominated one (C5), filtered and not --
    bit-exact against the oracle, and the instrumented stats confirm the path."""
    w = synth.make_config(name, scale=scale)
    pts = w.points[np.random.default_rng(11).permutation(w.n)]
    fec.set_instrumentation(True)
    try:
        got = run_gpu(fec, pts, w.d_th, w.min_size, w.max_size)
        assert fec.stats()["binning"] == 1
    finally:
        fec.set_instrumentation(False)
    assert_same(got, oracle.fec(pts, w.d_th, w.min_size, w.max_size), f"shuffled {name}@{scale}")
    assert_same(run_gpu(fec, pts, w.d_th), oracle.fec(pts, w.d_th), f"shuffled {name}@{scale} unfiltered")


@pytest.mark.parametrize("mn,mx", [(1, 10**9), (3, 40)])
def test_large_sparse_dominated_bucketed_relabel(fec, mn, mx):
    """Sparse-dominated clouds of >= 2^22 points take the bucketed relabel (the size filter
    applied in the bucket pass; a filter keeping every size reduces no counts): C5 at 4% (4.4M
    points, shuffled: the key-sort path), with a no-op and a real size filter."""
    w = synth.make_config("C5", scale=0.04)
    assert w.n >= 1 << 22
    assert_same(run_gpu(fec, w.points, w.d_th, mn, mx), oracle.fec(w.points, w.d_th, mn, mx), f"C5@0.04 [{mn},{mx}]")


def test_deterministic_repeats(fec):
    w = synth.make_config("C5", scale=0.01)
    first = run_gpu(fec, w.points, w.d_th)
    for _ in range(10):
        assert_same(run_gpu(fec, w.points, w.d_th), first, "repeat")


def test_permutation_changes_only_label_values(fec):
    w = synth.make_config("C2")
    perm = np.random.default_rng(3).permutation(w.n)
    a = run_gpu(fec, w.points, w.d_th)
    b = run_gpu(fec, w.points[perm], w.d_th)
    assert_same(b, oracle.fec(w.points[perm], w.d_th), "permuted")
    pairs = np.unique(np.stack([a[perm], b], 1), axis=0)
    assert len(np.unique(pairs[:, 0])) == len(pairs) == len(np.unique(pairs[:, 1]))


def test_edge_cases(fec):
    # n = 0, n = 1, all identical, a single huge cell, max_size below min component
    assert run_gpu(fec, np.zeros((0, 3), np.float32), 1.0).shape == (0,)
    assert_same(run_gpu(fec, np.array([[1, 2, 3]], np.float32), 0.5), np.array([0], np.int32), "n=1")
    same = np.full((5000, 3), -7.5, np.float32)
    assert_same(run_gpu(fec, same, 1e-3), np.zeros(5000, np.int32), "identical")
    assert_same(run_gpu(fec, same, 1e-3, 5001, 10**6), np.full(5000, -1, np.int32), "identical filtered")
    dense = np.random.default_rng(0).uniform(0, 0.2, size=(30000, 3)).astype(np.float32)
    assert_same(run_gpu(fec, dense, 0.25), oracle.fec(dense, 0.25), "one dense cell")
    # points exactly on cell boundaries, multiples of d (worst case for the grid)
    p, d, _ = synth.random_cloud(5, n=3000, geometry="cell_edges")
    assert_same(run_gpu(fec, p, d), oracle.fec(p, d), "cell edges")
    # a huge sparse bbox forces the hashed cell table
    rng = np.random.default_rng(1)
    sparse = np.concatenate([rng.uniform(0, 1, size=(2000, 3)),
                             rng.uniform(0, 1, size=(2000, 3)) + 50000.0]).astype(np.float32)
    fec.set_instrumentation(True)
    try:
        assert_same(run_gpu(fec, sparse, 0.1), oracle.fec(sparse, 0.1), "hashed table")
        assert fec.stats()["dense_table"] == 0
    finally:
        fec.set_instrumentation(False)


def test_error_paths_gpu(fec):
    p = np.random.default_rng(0).uniform(0, 1, size=(100, 3)).astype(np.float32)
    t = torch.from_numpy(p).cuda()
    out = torch.full((100,), 12345, dtype=torch.int32, device="cuda")
    for d in (0.0, -1.0, float("nan"), float("inf"), 1e-20, 1e20):
        with pytest.raises(fec.FecError) as e:
            fec.cluster(t, d, out=out)
        assert e.value.code == fec.ERR_INVALID_ARGUMENT
    assert (out == 12345).all()                 # untouched on argument errors
    with pytest.raises(fec.FecError) as e:
        fec.cluster(t, 0.1, 5, 4)
    assert e.value.code == fec.ERR_INVALID_ARGUMENT
    q = p.copy()
    q[37, 1] = np.nan
    with pytest.raises(fec.FecError) as e:
        fec.cluster(torch.from_numpy(q).cuda(), 0.1, out=out)
    assert e.value.code == fec.ERR_NONFINITE
    q[37, 1] = np.inf
    with pytest.raises(fec.FecError) as e:
        fec.cluster(torch.from_numpy(q).cuda(), 0.1)
    assert e.value.code == fec.ERR_NONFINITE
    assert (out == 12345).all()
    far = np.array([[0, 0, 0], [1e6, 0, 0]], np.float32)
    with pytest.raises(fec.FecError) as e:
        fec.cluster(torch.from_numpy(far).cuda(), 1e-3)
    assert e.value.code == fec.ERR_GRID_RANGE
    # a host pointer where a device pointer is required
    L = fec.lib()
    ws = torch.empty(fec.workspace_bytes(100), dtype=torch.uint8, device="cuda")
    rc = L.fec_cluster_ws(p.ctypes.data, 100, 0.1, 1, 10, out.data_ptr(), ws.data_ptr(), ws.numel(), None)
    assert rc == fec.ERR_INVALID_ARGUMENT
    rc = L.fec_cluster_ws(t.data_ptr(), 100, 0.1, 1, 10, out.data_ptr(), ws.data_ptr(), 10, None)
    assert rc == fec.ERR_INVALID_ARGUMENT


def test_instrumentation_counts(fec):
    w = synth.make_config("C1")
    fec.set_instrumentation(True)
    try:
        run_gpu(fec, w.points, w.d_th)
        s = fec.stats()
    finally:
        fec.set_instrumentation(False)
    un = oracle.fec(w.points, w.d_th)
    assert s["components"] == len(np.unique(un))
    assert 0 < s["cells"] <= w.n
    assert s["pair_tests"] > 0
    fec.set_grid_mode(1)
    fec.set_instrumentation(True)
    try:
        run_gpu(fec, w.points, w.d_th)
        h = fec.stats()
    finally:
        fec.set_instrumentation(False)
        fec.set_grid_mode(0)
    assert s["dense_table"] == 1 and h["dense_table"] == 0 and h["components"] == s["components"]
    assert h["cells"] == s["cells"] and h["dims"] == s["dims"]


@pytest.mark.parametrize("cap", [1, 7])
def test_uncertain_queue_overflow_path(fec, cap):
    """Dense cells: uncertain component pairs beyond the queue cap are tested in place by one
    thread; the labels must not change."""
    fec.set_item_cap(cap)
    try:
        for name, scale in [("C3", 0.02), ("C4", 0.01), ("C5", 0.005)]:
            w = synth.make_config(name, scale=scale)
            got = run_gpu(fec, w.points, w.d_th, 1, 2**62)
            assert_same(got, oracle.fec(w.points, w.d_th, 1, 2**62), f"{name} cap {cap}")
        rng = np.random.default_rng(11)
        for k in range(20):
            n = int(rng.integers(50, 3000))
            c = rng.uniform(0, 3, size=(6, 3))
            pts = (c[rng.integers(0, 6, n)] + rng.normal(0, 0.15, (n, 3))).astype(np.float32)
            d = float(rng.uniform(0.05, 0.4))
            got = run_gpu(fec, pts, d)
            assert_same(got, oracle.fec(pts, d, 1, 2**62), f"blobs {k} cap {cap}")
    finally:
        fec.set_item_cap(0)
