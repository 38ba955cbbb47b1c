"""The asynchronous boundary (SURVEY §8(b) fec_cluster_async): no host round trip, device-side
errors through status_dev, CUDA-graph capture and replay, the north-star signature
fec_cluster called directly through ctypes, and the forced-OOM hook.  Every label is compared
with the live oracle on the same seeded input (bit-exact)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fec():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2208_07678_b200 as fec
    fec.lib()
    return fec


def assert_same(got, want, ctx=""):
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{ctx}: {bad.size}/{want.size} labels differ; first {bad[:5]} "
                             f"got {got[bad[:5]]} want {want[bad[:5]]}")


def test_fec_cluster_north_star_signature(fec):
    """fec_cluster(points, n, d_th, min_size, max_size, labels_out) called directly (ctypes):
    self-allocating, synchronous, returns the device status."""
    L = fec.lib()
    for name in ("C1", "C2"):
        w = synth.make_config(name)
        x = torch.from_numpy(w.points).cuda()
        out = torch.full((w.n,), -5, dtype=torch.int32, device="cuda")
        rc = L.fec_cluster(x.data_ptr(), w.n, float(np.float32(w.d_th)), w.min_size, w.max_size, out.data_ptr())
        assert rc == fec.OK, L.fec_last_error()
        assert_same(out.cpu().numpy(), oracle.fec(w.points, w.d_th, w.min_size, w.max_size), name)
    for seed in range(12):
        p, d, geom = synth.random_cloud(seed)
        x = torch.from_numpy(p).cuda()
        out = torch.empty(len(p), dtype=torch.int32, device="cuda")
        assert L.fec_cluster(x.data_ptr(), len(p), d, 2, 500, out.data_ptr()) == fec.OK
        assert_same(out.cpu().numpy(), oracle.fec(p, d, 2, 500), f"seed {seed} {geom}")
    q = synth.make_config("C1").points.copy()
    q[123, 2] = np.nan
    x = torch.from_numpy(q).cuda()
    out = torch.full((len(q),), 77, dtype=torch.int32, device="cuda")
    assert L.fec_cluster(x.data_ptr(), len(q), 0.5, 1, 10, out.data_ptr()) == fec.ERR_NONFINITE
    assert (out == 77).all()
    assert L.fec_cluster(None, 0, 0.5, 1, 10, None) == fec.OK


def test_async_status_dev(fec):
    """Errors found on the device reach status_dev in stream order; labels stay untouched."""
    status = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    w = synth.make_config("C1")
    x = torch.from_numpy(w.points).cuda()
    out = torch.empty(w.n, dtype=torch.int32, device="cuda")
    fec.cluster_async(x, w.d_th, w.min_size, w.max_size, out, status)
    torch.cuda.synchronize()
    assert int(status.item()) == fec.OK
    assert_same(out.cpu().numpy(), oracle.fec(w.points, w.d_th, w.min_size, w.max_size), "C1 async")
    q = w.points.copy()
    q[5, 0] = np.inf
    out2 = torch.full((w.n,), 31, dtype=torch.int32, device="cuda")
    fec.cluster_async(torch.from_numpy(q).cuda(), w.d_th, 1, 10, out2, status)
    torch.cuda.synchronize()
    assert int(status.item()) == fec.ERR_NONFINITE and (out2 == 31).all()
    far = torch.tensor([[0, 0, 0], [1e6, 0, 0]], dtype=torch.float32, device="cuda")
    out3 = torch.full((2,), 31, dtype=torch.int32, device="cuda")
    fec.cluster_async(far, 1e-3, 1, 10, out3, status)
    torch.cuda.synchronize()
    assert int(status.item()) == fec.ERR_GRID_RANGE and (out3 == 31).all()


def _capture(fn):
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # warm-up outside the graph (library state, allocator)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        fn()
    torch.cuda.synchronize()
    return g


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_graph_capture_replays_bit_exact(fec, name):
    """fec_cluster_ws_async captured in a CUDA graph and replayed 10 times: every replay
    recomputes the labels from the current contents of the input buffer (the grid plan is
    made on the device), so replays on a different cloud of the same size are right too."""
    w = synth.make_config(name)
    want = oracle.fec(w.points, w.d_th, w.min_size, w.max_size)
    x = torch.from_numpy(w.points).cuda()
    out = torch.empty(w.n, dtype=torch.int32, device="cuda")
    ws = torch.empty(fec.workspace_bytes(w.n), dtype=torch.uint8, device="cuda")
    status = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    g = _capture(lambda: fec.cluster(x, w.d_th, w.min_size, w.max_size, out=out, workspace=ws, status=status,
                                     check=False))
    for k in range(10):
        out.fill_(-9)
        status.fill_(99)
        g.replay()
        torch.cuda.synchronize()
        assert int(status.item()) == fec.OK
        assert_same(out.cpu().numpy(), want, f"{name} replay {k}")
    # a different cloud (same n) in the same buffer: the replay re-plans on the device
    rng = np.random.default_rng(5)
    other = (w.points[rng.permutation(w.n)] * np.float32(1.5) + np.float32(3.0)).astype(np.float32)
    x.copy_(torch.from_numpy(other))
    g.replay()
    torch.cuda.synchronize()
    if w.n < 10**6:  # (the oracle on a second 27M-point cloud would double the test's CPU time)
        assert_same(out.cpu().numpy(), oracle.fec(other, w.d_th, w.min_size, w.max_size), f"{name} other cloud")
    # a NaN written into the captured input: the replay reports it and leaves the labels alone
    bad = other.copy()
    bad[w.n // 2, 1] = np.nan
    x.copy_(torch.from_numpy(bad))
    out.fill_(-9)
    g.replay()
    torch.cuda.synchronize()
    assert int(status.item()) == fec.ERR_NONFINITE and (out == -9).all()


def test_graph_capture_self_allocating(fec):
    """fec_cluster_async (stream-ordered workspace from the memory pool) inside a graph."""
    w = synth.make_config("C2")
    want = oracle.fec(w.points, w.d_th, w.min_size, w.max_size)
    x = torch.from_numpy(w.points).cuda()
    out = torch.empty(w.n, dtype=torch.int32, device="cuda")
    status = torch.full((1,), 99, dtype=torch.int32, device="cuda")
    g = _capture(lambda: fec.cluster_async(x, w.d_th, w.min_size, w.max_size, out, status))
    for k in range(10):
        out.fill_(-9)
        g.replay()
        torch.cuda.synchronize()
        assert int(status.item()) == fec.OK
        assert_same(out.cpu().numpy(), want, f"replay {k}")


def test_forced_out_of_memory(fec):
    L = fec.lib()
    w = synth.make_config("C1")
    x = torch.from_numpy(w.points).cuda()
    out = torch.full((w.n,), 3, dtype=torch.int32, device="cuda")
    fec.debug_alloc_extra(1 << 52)  # 4 PiB: no pool can serve it
    try:
        assert L.fec_cluster(x.data_ptr(), w.n, 0.5, 1, 10, out.data_ptr()) == fec.ERR_OUT_OF_MEMORY
        assert b"cudaMallocAsync" in L.fec_last_error()
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        with pytest.raises(fec.FecError) as e:
            fec.cluster_async(x, 0.5, 1, 10, out, st)
        assert e.value.code == fec.ERR_OUT_OF_MEMORY
    finally:
        fec.debug_alloc_extra(0)
    torch.cuda.synchronize()
    assert (out == 3).all()
    assert L.fec_cluster(x.data_ptr(), w.n, 0.5, 10, 10**6, out.data_ptr()) == fec.OK
    assert_same(out.cpu().numpy(), oracle.fec(w.points, 0.5, 10, 10**6), "after OOM")


def test_foreign_stream_ordering(fec):
    """A stream other than the current one: inputs produced on the current stream are awaited,
    and the result is valid in the given stream's order."""
    w = synth.make_config("C2")
    want = oracle.fec(w.points, w.d_th, w.min_size, w.max_size)
    s = torch.cuda.Stream()
    for _ in range(3):
        x = torch.from_numpy(w.points).cuda() * 1.0  # produced on the current stream
        lab = fec.cluster(x, w.d_th, w.min_size, w.max_size, stream=s, check=False)
        s.synchronize()
        assert_same(lab.cpu().numpy(), want, "foreign stream")


def test_debug_sync_flag_reports_nothing_on_a_clean_run(fec):
    """FEC_DEBUG_SYNC=1 (synchronise after every launch, name the failing kernel) on a clean run:
    same labels, no report."""
    import subprocess
    import sys
    code = ("import sys; sys.path.insert(0, '.'); import numpy as np, torch, synth, oracle; "
            "import paper_2208_07678_b200 as fec; w = synth.make_config('C2'); "
            "lab = fec.cluster(torch.from_numpy(w.points).cuda(), w.d_th, w.min_size, w.max_size).cpu().numpy(); "
            "assert np.array_equal(lab, oracle.fec(w.points, w.d_th, w.min_size, w.max_size)); print('ok')")
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600,
                       env={**os.environ, "FEC_DEBUG_SYNC": "1"})
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
    assert "FEC_DEBUG_SYNC" not in r.stderr
