"""GPU parity of the multi-GPU slab path through the C ABI (fec_slab_local / fec_slab_merge),
with the ranks emulated one after another in one process on one GPU (the kernels of one
rank never wait on another rank's, so this is the same code the N-GPU run executes; the
all-gather becomes a concatenation).  Bar: the union of the ranks' owned labels equals the
oracle on the whole cloud, bit for bit."""
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


def run_emulated(fec, pts, d, world, mn=1, mx=HUGE):
    from paper_2208_07678_b200 import dist as fdist
    plan = fdist.plan_slabs(pts, d, world)
    words = fec.slab_record_words(plan.rec_cap)
    shards, bufs = [], []
    for r in range(world):
        sh = fdist.shard(pts, plan, r)
        x = torch.from_numpy(sh.points).cuda()
        g = torch.from_numpy(sh.gidx).cuda()
        ws = torch.empty(fec.slab_workspace_bytes(sh.points.shape[0], world, plan.rec_cap), dtype=torch.uint8,
                         device="cuda")
        rec = torch.full((words,), -99, dtype=torch.int32, device="cuda")
        state = fec.slab_local(x, g, sh.n_owned, sh.n_first, d, rec, plan.rec_cap, ws)
        shards.append((sh, x, g, ws, state))
        bufs.append(rec)
    allrec = torch.cat(bufs)
    labels = np.full(pts.shape[0], -7, np.int32)
    for r, (sh, x, g, ws, state) in enumerate(shards):
        lab = torch.full((sh.n_owned,), -9, dtype=torch.int32, device="cuda")
        fec.slab_merge(allrec, world, r, mn, mx, lab, ws, state)
        torch.cuda.synchronize()
        labels[sh.gidx[:sh.n_owned]] = lab.cpu().numpy()
    return labels, plan


def assert_same(got, want, ctx):
    if not np.array_equal(got, want):
        bad = np.nonzero(got != want)[0]
        raise AssertionError(f"{ctx}: {bad.size}/{want.size} differ; first {bad[:5]} got {got[bad[:5]]} "
                             f"want {want[bad[:5]]}")


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_slab_random_clouds(fec, world):
    from test_dist_cpu import clouds
    for k, (pts, d) in enumerate(clouds()):
        for mn, mx in [(1, HUGE), (10, 300)]:
            got, _ = run_emulated(fec, pts, d, world, mn, mx)
            assert_same(got, oracle.fec(pts, d, mn, mx), f"cloud {k} world {world} [{mn},{mx}]")


@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C2", 1.0), ("C3", 0.05), ("C4", 0.02), ("C5", 0.01)])
@pytest.mark.parametrize("world", [2, 8])
def test_slab_configs(fec, name, scale, world):
    w = synth.make_config(name, scale=scale)
    for mn, mx in [(w.min_size, w.max_size), (1, HUGE)]:
        got, plan = run_emulated(fec, w.points, w.d_th, world, mn, mx)
        assert_same(got, oracle.fec(w.points, w.d_th, mn, mx), f"{name}x{scale} world {world}")


def test_slab_world1_equals_single(fec):
    w = synth.make_config("C1")
    got, _ = run_emulated(fec, w.points, w.d_th, 1, w.min_size, w.max_size)
    t = torch.from_numpy(w.points).cuda()
    single = fec.cluster(t, w.d_th, w.min_size, w.max_size).cpu().numpy()
    assert_same(got, single, "world 1")


def test_slab_giant_component_across_all_slabs(fec):
    # a dense chain along x joins every slab into one component; sizes sum over ranks
    rng = np.random.default_rng(3)
    x = np.sort(rng.uniform(0, 40, 20000)).astype(np.float32)
    pts = np.stack([x, rng.uniform(0, 0.2, x.size), rng.uniform(0, 0.2, x.size)], 1).astype(np.float32)
    perm = rng.permutation(x.size)
    pts = pts[perm]
    for world in (2, 5, 8):
        for mn, mx in [(1, HUGE), (20001, HUGE), (1, 19999), (20000, 20000)]:
            got, _ = run_emulated(fec, pts, 0.3, world, mn, mx)
            assert_same(got, oracle.fec(pts, 0.3, mn, mx), f"chain world {world} [{mn},{mx}]")


def test_slab_edge_cases(fec):
    # more ranks than occupied layers (trailing empty slabs), single point, empty cloud
    for pts in (np.array([[0, 0, 0], [0.1, 0, 0], [5, 0, 0]], np.float32),
                np.array([[1, 2, 3]], np.float32),
                np.zeros((0, 3), np.float32)):
        for world in (2, 4, 8):
            got, _ = run_emulated(fec, pts, 0.2, world)
            assert_same(got, oracle.fec(pts, 0.2, 1, HUGE), f"edge n={len(pts)} world {world}")


def test_slab_argument_errors(fec):
    x = torch.zeros((4, 3), dtype=torch.float32, device="cuda")
    g = torch.arange(4, dtype=torch.int32, device="cuda")
    rec = torch.zeros(fec.slab_record_words(4), dtype=torch.int32, device="cuda")
    ws = torch.empty(fec.slab_workspace_bytes(4, 2, 4), dtype=torch.uint8, device="cuda")
    with pytest.raises(fec.FecError):
        fec.slab_local(x, g, 2, 3, 0.5, rec, 4, ws)   # n_first > n_owned
    with pytest.raises(fec.FecError):
        fec.slab_local(x, g, 2, 1, 0.5, rec, 2, ws)   # rec_cap < boundary points (1 + 2)
    st = fec.slab_local(x, g, 2, 1, 0.5, rec, 4, ws)
    lab = torch.empty(2, dtype=torch.int32, device="cuda")
    allrec = torch.cat([rec, rec])
    with pytest.raises(fec.FecError):
        fec.slab_merge(allrec, 2, 2, 1, 10, lab, ws, st)  # rank >= world
    with pytest.raises(fec.FecError):
        fec.slab_merge(allrec, 2, 0, 1, 10, lab, ws, fec.SlabState())  # state not filled


def run_mode_b_emulated(fec, pts, d, world):
    """Mode B with the ranks emulated on one GPU: fec_part_* per rank, the collectives replaced
    by their definitions (min / sum / exchange of the packed segments)."""
    from paper_2208_07678_b200 import dist as fdist
    n = pts.shape[0]
    ranks = []
    for r in range(world):
        lo, hi = (n * r) // world, (n * (r + 1)) // world
        ops = fdist.DevicePartOps("cuda")
        ranks.append((ops, torch.from_numpy(pts[lo:hi].copy()).cuda(), torch.arange(lo, hi, dtype=torch.int32, device="cuda")))
    bbs = [ops.bbox(p) for ops, p, _ in ranks]
    gbb = torch.stack(bbs).min(0).values
    hists = [ops.hist(p, gbb, d) for ops, p, _ in ranks]
    ghist = torch.stack([h.to(torch.int64) for h in hists]).sum(0).to(torch.int32)
    plans = [ops.plan(ghist, world) for ops, _, _ in ranks]
    for pl in plans[1:]:
        assert torch.equal(pl, plans[0])
    rec_cap = int(plans[0][4 * world + 1].item())
    sends = []
    for (ops, p, g), pl in zip(ranks, plans):
        c = ops.count(p, g, gbb, d, pl, world)
        sp, sg = ops.pack(p, g, gbb, d, pl, world, c, int(c.sum().item()))
        sends.append((c.cpu().tolist(), sp, sg))
    out = []
    for r, ((ops, _, _), pl) in enumerate(zip(ranks, plans)):
        rp, rg = [], []
        for c, sp, sg in sends:
            o = sum(c[:r])
            rp.append(sp[o:o + c[r]])
            rg.append(sg[o:o + c[r]])
        op, og, c3 = ops.order(torch.cat(rp), torch.cat(rg), gbb, d, pl, world, r)
        c3 = c3.cpu().tolist()
        out.append(fdist.Shard(op, og, int(c3[0] + c3[1]), int(c3[0])))
    return out, rec_cap


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_mode_b_partition_equals_planner(fec, world):
    """The device partition (fec_part_*) gives every rank exactly the host planner's slab (owned,
    first layer, halo), and Mode A on those slabs equals the oracle on the whole cloud."""
    from paper_2208_07678_b200 import dist as fdist
    from test_dist_cpu import clouds, _same_slab
    cases = list(clouds()) + [(synth.make_config("C2").points, 0.35),
                              (synth.make_config("C4", scale=0.01).points, 0.25)]
    for k, (pts, d) in enumerate(cases):
        shards, rec_cap = run_mode_b_emulated(fec, pts, d, world)
        plan = fdist.plan_slabs(pts, d, world)
        assert rec_cap == plan.rec_cap, (k, rec_cap, plan.rec_cap)
        for r, sh in enumerate(shards):
            sh_h = fdist.Shard(sh.points.cpu().numpy(), sh.gidx.cpu().numpy(), sh.n_owned, sh.n_first)
            assert _same_slab(sh_h, fdist.shard(pts, plan, r)), (k, world, r)
        # Mode A on the device-partitioned slabs
        words = fec.slab_record_words(rec_cap)
        states, bufs, wss = [], [], []
        for sh in shards:
            ws = torch.empty(fec.slab_workspace_bytes(sh.points.shape[0], world, rec_cap), dtype=torch.uint8,
                             device="cuda")
            rec = torch.zeros(words, dtype=torch.int32, device="cuda")
            states.append(fec.slab_local(sh.points, sh.gidx, sh.n_owned, sh.n_first, d, rec, rec_cap, ws))
            bufs.append(rec)
            wss.append(ws)
        allrec = torch.cat(bufs)
        labels = np.full(pts.shape[0], -7, np.int32)
        for r, sh in enumerate(shards):
            lab = torch.full((sh.n_owned,), -9, dtype=torch.int32, device="cuda")
            fec.slab_merge(allrec, world, r, 1, HUGE, lab, wss[r], states[r])
            torch.cuda.synchronize()
            labels[sh.gidx[:sh.n_owned].cpu().numpy()] = lab.cpu().numpy()
        assert_same(labels, oracle.fec(pts, d, 1, HUGE), f"mode B case {k} world {world}")
