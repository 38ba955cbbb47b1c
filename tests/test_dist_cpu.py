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
