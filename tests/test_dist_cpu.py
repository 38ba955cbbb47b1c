"""Multi-GPU slab decomposition, host side (no GPU): plan/shard invariants, the record
protocol (modelled in numpy around the oracle's local clustering) and the all-gather
plumbing of paper_2208_07678_b200.dist over a world-size-2 `gloo` process group.

The CUDA kernels of the same protocol (fec_slab_local / fec_slab_merge) are checked on the
GPU in test_gpu_dist.py; here the model of those two steps is written from the protocol in
include/fec.h, so a wrong decomposition (a missed cross-slab edge, a double-counted halo
point, a wrong global size or minimum) fails against the oracle on the whole cloud."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2208_07678_b200 import dist as fdist

HUGE = 2**62


def clouds():
    rng = np.random.default_rng(7)
    out = []
    # long thin clouds so slabs have several layers; blobs crossing cut planes
    for k in range(6):
        n = int(rng.integers(200, 1500))
        p = rng.uniform([0, 0, 0], [12, 2, 2], size=(n, 3))
        if k % 2:
            c = rng.uniform([0, 0, 0], [12, 2, 2], size=(5, 3))
            p = np.concatenate([p, c[rng.integers(0, 5, n)] + rng.normal(0, 0.3, (n, 3))])
        out.append((p.astype(np.float32), float(rng.uniform(0.15, 0.6))))
    # points exactly on cell layers (dyadic spacing) and a chain crossing every cut
    x = np.arange(0, 64, dtype=np.float32) * np.float32(0.5)
    out.append((np.stack([x, np.zeros_like(x), np.zeros_like(x)], 1), 0.5))
    # tiny cloud: more ranks than layers
    out.append((np.array([[0, 0, 0], [0.1, 0, 0], [5, 0, 0]], np.float32), 0.2))
    return out


# ---- numpy model of fec_slab_local / fec_slab_merge (protocol of include/fec.h) ----------
HDR = 4


def c_off(rec_cap):
    return HDR + 2 * ((rec_cap + 1) // 2 * 2)


def words_of(rec_cap):
    return c_off(rec_cap) + 4 * rec_cap


def model_local(sh: fdist.Shard, d_th: float, rec_cap: int) -> np.ndarray:
    n = sh.points.shape[0]
    rec = np.zeros(words_of(rec_cap), np.int32)
    if n == 0:
        return rec
    root = oracle.fec(sh.points, d_th, 1, HUGE).astype(np.int64)  # local min index = root id
    bnd = np.zeros(n, bool)
    bnd[:sh.n_first] = True
    bnd[sh.n_owned:] = True
    size, mn, key = {}, {}, {}
    for i in range(n):
        r = int(root[i])
        if i < sh.n_owned:
            size[r] = size.get(r, 0) + 1
            mn[r] = min(mn.get(r, 2**31 - 1), int(sh.gidx[i]))
        if bnd[i]:
            key[r] = max(key.get(r, -1), int(sh.gidx[i]))
    P = [(int(sh.gidx[i]), key[int(root[i])]) for i in range(n) if bnd[i]]
    C = [(k, size.get(r, 0), mn.get(r, 2**31 - 1), r) for r, k in key.items()]
    rec[0], rec[1] = len(P), len(C)
    for j, (a, b) in enumerate(P):
        rec[HDR + 2 * j: HDR + 2 * j + 2] = (a, b)
    for j, c in enumerate(C):
        o = c_off(rec_cap) + 4 * j
        rec[o:o + 4] = c
    model_local.state = (root, size, mn)
    return rec


def model_merge(allrec: np.ndarray, world: int, rank: int, rec_cap: int, sh: fdist.Shard, state, mn_sz, mx_sz):
    words = words_of(rec_cap)
    par = {}

    def find(x):
        par.setdefault(x, x)
        while par[x] != x:
            par[x] = par[par[x]]
            x = par[x]
        return x

    for rk in range(world):
        r = allrec[rk * words:(rk + 1) * words]
        for j in range(r[0]):
            a, b = find(int(r[HDR + 2 * j])), find(int(r[HDR + 2 * j + 1]))
            if a != b:
                par[max(a, b)] = min(a, b)
    gs, gm = {}, {}
    for rk in range(world):
        r = allrec[rk * words:(rk + 1) * words]
        for j in range(r[1]):
            k, s, m, _ = r[c_off(rec_cap) + 4 * j: c_off(rec_cap) + 4 * j + 4]
            g = find(int(k))
            gs[g] = gs.get(g, 0) + int(s)
            gm[g] = min(gm.get(g, 2**31 - 1), int(m))
    if sh.n_owned == 0:
        return np.zeros(0, np.int32)
    root, size, mn = state
    size, mn = dict(size), dict(mn)
    own = allrec[rank * words:(rank + 1) * words]
    for j in range(own[1]):
        k, _, _, lr = own[c_off(rec_cap) + 4 * j: c_off(rec_cap) + 4 * j + 4]
        g = find(int(k))
        size[int(lr)], mn[int(lr)] = gs[g], gm[g]
    out = np.empty(sh.n_owned, np.int32)
    for i in range(sh.n_owned):
        r = int(root[i])
        out[i] = mn[r] if mn_sz <= size[r] <= mx_sz else -1
    return out


def run_model(pts, d, world, mn_sz=1, mx_sz=HUGE):
    plan = fdist.plan_slabs(pts, d, world)
    shards = [fdist.shard(pts, plan, r) for r in range(world)]
    recs, states = [], []
    for sh in shards:
        recs.append(model_local(sh, d, plan.rec_cap))
        states.append(getattr(model_local, "state", None))
    allrec = np.concatenate(recs)
    labels = np.full(pts.shape[0], -7, np.int32)
    for r, sh in enumerate(shards):
        lab = model_merge(allrec, world, r, plan.rec_cap, sh, states[r], mn_sz, mx_sz)
        labels[sh.gidx[:sh.n_owned]] = lab
    return labels


@pytest.mark.parametrize("world", [1, 2, 3, 5, 8])
def test_plan_covers_every_edge_once(world):
    for pts, d in clouds():
        plan = fdist.plan_slabs(pts, d, world)
        shards = [fdist.shard(pts, plan, r) for r in range(world)]
        owner = np.full(pts.shape[0], -1)
        for r, sh in enumerate(shards):
            own = sh.gidx[:sh.n_owned]
            assert (owner[own] == -1).all(), "point owned twice"
            owner[own] = r
            assert plan.rec_cap >= sh.n_first + (len(sh.gidx) - sh.n_owned)
            # the halo of rank r is exactly the first layer of the next non-empty rank
            halo = set(sh.gidx[sh.n_owned:].tolist())
            nxt = next((s for s in shards[r + 1:] if s.n_owned), None)
            assert halo == (set(nxt.gidx[:nxt.n_first].tolist()) if nxt else set())
        assert (owner >= 0).all(), "point owned by nobody"
        # every pred-true pair lies in some rank's owned ∪ halo
        i, j = oracle.brute.edges(pts, d)
        local = [set(sh.gidx.tolist()) for sh in shards]
        for a, b in zip(i.tolist(), j.tolist()):
            assert any(a in L and b in L for L in local), f"edge {a}-{b} seen by no rank"


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_record_protocol_model_equals_oracle(world):
    for pts, d in clouds():
        for mn_sz, mx_sz in [(1, HUGE), (10, 300), (3, 40)]:
            got = run_model(pts, d, world, mn_sz, mx_sz)
            want = oracle.fec(pts, d, mn_sz, mx_sz)
            np.testing.assert_array_equal(got, want)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = True
        for pts, d in clouds():
            plan = fdist.plan_slabs(pts, d, world)  # every rank plans the same cuts
            sh = fdist.shard(pts, plan, rank)
            rec = model_local(sh, d, plan.rec_cap)
            state = getattr(model_local, "state", None)
            allrec = fdist.exchange_records(torch.from_numpy(rec), world).numpy()
            lab = model_merge(allrec, world, rank, plan.rec_cap, sh, state, 10, HUGE)
            parts = [None] * world
            dist.all_gather_object(parts, (sh.gidx[:sh.n_owned], lab))
            if rank == 0:
                full = np.full(pts.shape[0], -7, np.int32)
                for g, l in parts:
                    full[g] = l
                ok &= bool(np.array_equal(full, oracle.fec(pts, d, 10, HUGE)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_exchange():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(240)
        assert p.exitcode == 0
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res[0] and res[1]


# ---- Mode B (device slab partition of index-sharded input), modelled in numpy ----------------
MAXL = 1 << 20  # fec_part_max_layers()


class NumpyPartOps:
    """numpy model of the fec_part_* steps (include/fec.h "Multi-GPU Mode B"), on CPU tensors, so
    dist.repartition's collectives run over gloo.  The layer arithmetic is the planner's:
    floor((x - lo) * (1/(c/2))) >> 1 in fp64, c = fp32(d)(1 + 2^-16)."""

    def bbox(self, points):
        import torch
        p = points.numpy()
        bad = not np.isfinite(p).all()
        if p.shape[0]:
            mn, mx = p.min(0), p.max(0)
        else:
            mn = np.full(3, np.finfo(np.float32).max, np.float32)
            mx = -mn
        return torch.from_numpy(np.concatenate([mn, -mx, [-1.0 if bad else 0.0, 0.0]]).astype(np.float32))

    @staticmethod
    def _axis(gbb, d):
        ext = (-gbb[3:6].astype(np.float64)) - gbb[:3].astype(np.float64)
        axis = int(np.argmax(ext))
        lo = np.float64(gbb[axis])
        inv_h = 1.0 / (fdist.cell_edge(d) * 0.5)
        nl = (int(np.floor((np.float64(-gbb[3 + axis]) - lo) * inv_h)) >> 1) + 1
        return axis, lo, inv_h, nl

    def _layers(self, p, gbb, d):
        axis, lo, inv_h, nl = self._axis(gbb, d)
        return (np.floor((p[:, axis].astype(np.float64) - lo) * inv_h).astype(np.int64) >> 1), nl

    def hist(self, points, gbb, d):
        import torch
        lay, nl = self._layers(points.numpy(), gbb.numpy(), d)
        return torch.from_numpy(np.bincount(lay, minlength=MAXL)[:MAXL].astype(np.int32))

    def plan(self, ghist, world):
        import torch
        hist = ghist.numpy().astype(np.int64)
        nl = int(np.nonzero(hist)[0].max()) + 1 if hist.any() else 1
        self._nl = nl
        cum = np.concatenate([[0], np.cumsum(hist[:nl])])
        n = int(cum[-1])
        cuts = np.zeros(world + 1, np.int64)
        cuts[world] = nl
        for r in range(1, world):
            b = int(np.searchsorted(cum, (n * r) // world, side="left"))
            cuts[r] = min(max(b, int(cuts[r - 1]) + 1), nl)
        owned = cum[cuts[1:]] - cum[cuts[:-1]]
        first = np.array([hist[cuts[r]] if (r > 0 and cuts[r] < nl) else 0 for r in range(world)], np.int64)
        halo = np.array([hist[cuts[r + 1]] if (cuts[r + 1] < nl and cuts[r + 1] > cuts[r]) else 0
                         for r in range(world)], np.int64)
        first[owned == 0] = 0
        halo[owned == 0] = 0
        rec = int((first + halo).max()) if world > 1 else 0
        return torch.from_numpy(np.concatenate([cuts, owned, first, halo, [rec, 0]]).astype(np.int64))

    def _dest(self, p, gbb, d, plan, world):
        lay, _ = self._layers(p, gbb.numpy(), d)
        pl = plan.numpy()
        cuts, owned = pl[:world + 1], pl[world + 1:2 * world + 1]
        r = np.searchsorted(cuts[1:world], lay, side="right")  # last r with cuts[r] <= L
        halo = (r > 0) & (lay == cuts[np.maximum(r, 0)]) & (owned[np.maximum(r - 1, 0)] > 0)
        return r, halo

    def count(self, points, gidx, gbb, d, plan, world):
        import torch
        r, halo = self._dest(points.numpy(), gbb, d, plan, world)
        c = np.bincount(r, minlength=world) + np.bincount(r[halo] - 1, minlength=world)
        return torch.from_numpy(c.astype(np.int64))

    def pack(self, points, gidx, gbb, d, plan, world, counts, total):
        import torch
        p, g = points.numpy(), gidx.numpy()
        r, halo = self._dest(p, gbb, d, plan, world)
        dst = np.concatenate([r, r[halo] - 1])
        src = np.concatenate([np.arange(len(p)), np.nonzero(halo)[0]])
        o = np.argsort(dst, kind="stable")
        return torch.from_numpy(p[src[o]].copy()), torch.from_numpy(g[src[o]].copy())

    def order(self, rpts, rgidx, gbb, d, plan, world, rank):
        import torch
        p, g = rpts.numpy(), rgidx.numpy()
        lay, _ = self._layers(p, gbb.numpy(), d)
        cuts = plan.numpy()[:world + 1]
        cat = np.where(lay >= cuts[rank + 1], 2, np.where((rank > 0) & (lay == cuts[rank]), 0, 1))
        o = np.argsort(cat, kind="stable")
        c3 = np.bincount(cat, minlength=3).astype(np.int64)
        return torch.from_numpy(p[o].copy()), torch.from_numpy(g[o].copy()), torch.from_numpy(c3)


def _same_slab(sh_b, sh_a):
    """Mode B's slab equals the host planner's: same owned / first-layer / halo point sets."""
    gb = sh_b.gidx.numpy() if hasattr(sh_b.gidx, "numpy") else sh_b.gidx
    ga = sh_a.gidx
    return (sh_b.n_owned == sh_a.n_owned and sh_b.n_first == sh_a.n_first and
            set(gb[:sh_b.n_first].tolist()) == set(ga[:sh_a.n_first].tolist()) and
            set(gb[sh_b.n_first:sh_b.n_owned].tolist()) == set(ga[sh_a.n_first:sh_a.n_owned].tolist()) and
            set(gb[sh_b.n_owned:].tolist()) == set(ga[sh_a.n_owned:].tolist()))


def _worker_mode_b(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ok = True
        for pts, d in clouds():
            n = pts.shape[0]
            lo, hi = (n * rank) // world, (n * (rank + 1)) // world  # index-range shard
            sh, rec_cap = fdist.repartition(torch.from_numpy(pts[lo:hi].copy()),
                                            torch.arange(lo, hi, dtype=torch.int32), d, ops=NumpyPartOps())
            plan = fdist.plan_slabs(pts, d, world)
            ok &= rec_cap == plan.rec_cap and _same_slab(sh, fdist.shard(pts, plan, rank))
            # then the Mode A protocol on the received slab, against the oracle on the whole cloud
            sh_np = fdist.Shard(sh.points.numpy(), sh.gidx.numpy(), sh.n_owned, sh.n_first)
            rec = model_local(sh_np, d, rec_cap)
            state = getattr(model_local, "state", None)
            allrec = fdist.exchange_records(torch.from_numpy(rec), world).numpy()
            lab = model_merge(allrec, world, rank, rec_cap, sh_np, state, 1, HUGE)
            parts = [None] * world
            dist.all_gather_object(parts, (sh_np.gidx[:sh_np.n_owned], lab))
            if rank == 0:
                full = np.full(n, -7, np.int32)
                for g, l in parts:
                    full[g] = l
                ok &= bool(np.array_equal(full, oracle.fec(pts, d, 1, HUGE)))
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


def test_mode_b_model_matches_planner_single_process():
    # world 1..5 emulated by hand (the model's collectives are elementwise min / sum / concat)
    ops = NumpyPartOps()
    import torch
    for world in (1, 2, 3, 5):
        for pts, d in clouds():
            n = pts.shape[0]
            shards = [(torch.from_numpy(pts[(n * r) // world:(n * (r + 1)) // world].copy()),
                       torch.arange((n * r) // world, (n * (r + 1)) // world, dtype=torch.int32)) for r in range(world)]
            bb = torch.stack([ops.bbox(p) for p, _ in shards]).min(0).values
            hist = sum(ops.hist(p, bb, d).to(torch.int64) for p, _ in shards).to(torch.int32)
            plan = ops.plan(hist, world)
            ref = fdist.plan_slabs(pts, d, world)
            assert np.array_equal(plan.numpy()[:world + 1][:len(ref.cuts)], ref.cuts)
            sends = [ops.pack(p, g, bb, d, plan, world, None, 0) for p, g in shards]
            dests = [ops._dest(p.numpy(), bb, d, plan, world) for p, _ in shards]
            for r in range(world):
                rp, rg = [], []
                for (sp, sg), (dr, halo) in zip(sends, dests):
                    dst = np.sort(np.concatenate([dr, dr[halo] - 1]), kind="stable")
                    rp.append(sp.numpy()[dst == r])
                    rg.append(sg.numpy()[dst == r])
                op, og, c3 = ops.order(torch.from_numpy(np.concatenate(rp)), torch.from_numpy(np.concatenate(rg)),
                                       bb, d, plan, world, r)
                sh = fdist.Shard(op, og, int(c3[0] + c3[1]), int(c3[0]))
                assert _same_slab(sh, fdist.shard(pts, ref, r)), (world, r)


def test_gloo_world2_mode_b():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker_mode_b, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
        assert p.exitcode == 0
    res = dict(q.get(timeout=5) for _ in range(2))
    assert res[0] and res[1]
