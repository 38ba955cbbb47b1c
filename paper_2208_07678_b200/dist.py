"""Multi-GPU driver of the FEC path: spatial slabs, one all-gather, replicated merge.

SURVEY §8(e).  PAPER.md's FEC is a serial CPU loop (L480 names a parallel version as future
work), so the decomposition is this library's own:

* ``plan_slabs`` (host, setup — the cloud "is sharded … into spatial slabs" before the timed
  region, BASELINE.json north_star): cut the longest bbox axis into count-balanced slabs on
  boundaries of a grid whose cell edge is ``c = d_th*(1+2^-16)`` (> d_th, reading A6), so an
  edge of Eq. 1's graph only joins points of the same or adjacent cell
  layers.  Rank r owns layers [B_r, B_{r+1}) and holds, as a halo, layer B_{r+1} (the first
  layer of rank r+1): every cross-slab edge then lies inside exactly one rank's owned ∪ halo.
* ``shard``: the local input of one rank in the order the C ABI expects
  (first-layer owned | other owned | halo) with global indices.
* ``cluster_sharded`` (the timed step): ``fec_slab_local`` → ``exchange_records`` (NCCL
  ``all_gather_into_tensor`` over NVLink) → ``fec_slab_merge``.  All arithmetic runs in
  libfec.so's kernels; this module only moves buffers.

The labels a rank returns are global: minimum global index of the point's component over
the whole cloud, or -1 when the component's total size is outside [min_size, max_size].
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import slab_local, slab_merge, slab_record_words, slab_workspace_bytes, _f32


def cell_edge(d_th: float) -> float:
    """Slab grid cell edge: c = fp32(d_th) * (1 + 2^-16) in fp64 (reading A6)."""
    return float(np.float32(d_th)) * (1.0 + 2.0 ** -16)


@dataclass
class SlabPlan:
    world: int
    axis: int            # cut axis (longest bbox extent; ties -> lowest axis)
    lo: float            # bbox minimum along the axis (fp32 value)
    c: float             # cell edge (fp64)
    cuts: np.ndarray     # int64 [world+1]: rank r owns cell layers [cuts[r], cuts[r+1])
    rec_cap: int         # record capacity, the same on every rank
    n_owned: np.ndarray  # int64 [world]
    n_first: np.ndarray  # int64 [world]: owned points in layer cuts[r] (0 for rank 0)
    n_halo: np.ndarray   # int64 [world]: points in layer cuts[r+1] held by rank r


def cell_layers(points: np.ndarray, axis: int, lo: float, c: float) -> np.ndarray:
    """floor((x - lo) / c) along `axis`, in fp64 (x, lo are fp32 values)."""
    x = points[:, axis].astype(np.float64)
    return np.floor((x - np.float64(lo)) * (1.0 / c)).astype(np.int64)


def plan_slabs(points: np.ndarray, d_th: float, world: int) -> SlabPlan:
    """Count-balanced slab cuts on cell-layer boundaries (host; setup, not the timed step).

    Slabs are non-empty and at least one layer thick while there are enough layers; if the
    cloud has fewer occupied layers than ranks, the trailing ranks get empty slabs."""
    pts = np.asarray(points, dtype=np.float32).reshape(-1, 3)
    n = pts.shape[0]
    if world < 1:
        raise ValueError("world must be >= 1")
    c = cell_edge(d_th)
    if n == 0:
        z = np.zeros(world, np.int64)
        return SlabPlan(world, 0, 0.0, c, np.zeros(world + 1, np.int64), 0, z, z.copy(), z.copy())
    ext = pts.max(axis=0).astype(np.float64) - pts.min(axis=0).astype(np.float64)
    axis = int(np.argmax(ext))
    lo = float(pts[:, axis].min())
    lay = cell_layers(pts, axis, lo, c)
    nl = int(lay.max()) + 1
    hist = np.bincount(lay, minlength=nl).astype(np.int64)
    cum = np.concatenate([[0], np.cumsum(hist)])  # cum[k] = points in layers < k
    cuts = np.zeros(world + 1, np.int64)
    cuts[world] = nl
    for r in range(1, world):
        target = (n * r) // world
        b = int(np.searchsorted(cum, target, side="left"))  # first k with cum[k] >= target
        b = max(b, int(cuts[r - 1]) + 1)                      # at least one layer per slab
        cuts[r] = min(b, nl)
    owned = cum[cuts[1:]] - cum[cuts[:-1]]
    first = np.array([hist[cuts[r]] if (r > 0 and cuts[r] < nl) else 0 for r in range(world)], np.int64)
    halo = np.array([hist[cuts[r + 1]] if (cuts[r + 1] < nl and cuts[r + 1] > cuts[r]) else 0
                     for r in range(world)], np.int64)
    # a slab without points holds nothing (not even a halo); its neighbours are >= 2 layers apart
    first[owned == 0] = 0
    halo[owned == 0] = 0
    rec_cap = int((first + halo).max()) if world > 1 else 0
    return SlabPlan(world, axis, lo, c, cuts, rec_cap, owned, first, halo)


@dataclass
class Shard:
    points: np.ndarray   # float32 [n_local, 3]: first-layer owned | other owned | halo
    gidx: np.ndarray     # int32 [n_local]: global input index of each local point
    n_owned: int
    n_first: int


def shard(points: np.ndarray, plan: SlabPlan, rank: int) -> Shard:
    """Rank `rank`'s local input (owned points keep increasing global order inside each part)."""
    pts = np.asarray(points, dtype=np.float32).reshape(-1, 3)
    if pts.shape[0] == 0 or plan.n_owned[rank] == 0:
        return Shard(np.zeros((0, 3), np.float32), np.zeros(0, np.int32), 0, 0)
    lay = cell_layers(pts, plan.axis, plan.lo, plan.c)
    b0, b1 = int(plan.cuts[rank]), int(plan.cuts[rank + 1])
    first = np.flatnonzero(lay == b0) if rank > 0 else np.zeros(0, np.int64)
    rest = np.flatnonzero((lay >= b0) & (lay < b1) & ((lay != b0) if rank > 0 else True))
    halo = np.flatnonzero(lay == b1) if b1 < int(lay.max()) + 1 else np.zeros(0, np.int64)
    g = np.concatenate([first, rest, halo]).astype(np.int32)
    sh = Shard(pts[g], g, len(first) + len(rest), len(first))
    assert sh.n_owned == plan.n_owned[rank] and sh.n_first == plan.n_first[rank]
    assert len(halo) == plan.n_halo[rank]
    return sh


def exchange_records(send, world: int, group=None):
    """The one collective of the path: all-gather every rank's record buffer (rank r's at
    offset r).  NCCL over NVLink/NVSwitch on GPUs; any torch.distributed backend works."""
    import torch
    import torch.distributed as dist
    recv = torch.empty(world * send.numel(), dtype=send.dtype, device=send.device)
    if world == 1:
        recv.copy_(send)
    elif send.is_cuda and dist.get_backend(group) == "gloo":
        # test plumbing only (several ranks sharing one GPU): gloo gathers host tensors
        host = torch.empty(world * send.numel(), dtype=send.dtype)
        dist.all_gather_into_tensor(host, send.cpu(), group=group)
        recv.copy_(host)
    else:
        dist.all_gather_into_tensor(recv, send, group=group)
    return recv


class SlabRunner:
    """Device buffers of one rank, allocated once; ``step()`` is the timed multi-GPU step."""

    def __init__(self, points, gidx, n_owned: int, n_first: int, rec_cap: int, d_th: float, min_size: int,
                 max_size: int, world: int, rank: int, group=None):
        import torch
        self.points, self.gidx = points, gidx
        self.n_owned, self.n_first, self.rec_cap = int(n_owned), int(n_first), int(rec_cap)
        self.d_th, self.min_size, self.max_size = _f32(d_th), int(min_size), int(max_size)
        self.world, self.rank, self.group = int(world), int(rank), group
        dev = points.device
        words = slab_record_words(rec_cap)
        self.send = torch.empty(words, dtype=torch.int32, device=dev)
        self.labels = torch.empty(self.n_owned, dtype=torch.int32, device=dev)
        nb = slab_workspace_bytes(points.shape[0], world, rec_cap)
        self.ws = torch.empty(nb, dtype=torch.uint8, device=dev)
        self.recv = None

    def step(self):
        state = slab_local(self.points, self.gidx, self.n_owned, self.n_first, self.d_th, self.send, self.rec_cap,
                           self.ws)
        self.recv = exchange_records(self.send, self.world, self.group)
        slab_merge(self.recv, self.world, self.rank, self.min_size, self.max_size, self.labels, self.ws, state)
        return self.labels


def cluster_sharded(points, gidx, n_owned: int, n_first: int, d_th: float, min_size: int, max_size: int,
                    rec_cap: int, group=None):
    """One rank's part of a multi-GPU clustering (collective over `group`).  Returns int32
    labels of the rank's owned points (local order), valued in global indices."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    return SlabRunner(points, gidx, n_owned, n_first, rec_cap, d_th, min_size, max_size, world, rank,
                      group).step()


# ---- Mode B: index-sharded input -> spatial slabs on the device ----------
class DevicePartOps:
    """The steps of Mode B in libfec.so (fec_part_*, include/fec.h), on one device."""

    def __init__(self, device):
        import torch
        from . import lib
        self.L = lib()
        self.dev = torch.device(device)
        self.ws = torch.empty(int(self.L.fec_part_workspace_bytes()), dtype=torch.uint8, device=self.dev)
        self.nl = int(self.L.fec_part_max_layers())

    def _st(self):
        import torch
        return torch.cuda.current_stream(self.dev).cuda_stream

    def _chk(self, rc):
        from . import _check
        _check(rc)

    @staticmethod
    def _p(t):
        return t.data_ptr() if t is not None and t.numel() else None

    def bbox(self, points):
        import torch
        out = torch.empty(8, dtype=torch.float32, device=self.dev)
        self.hist_buf = torch.empty(self.nl, dtype=torch.int32, device=self.dev)
        self._chk(self.L.fec_part_bbox(self._p(points), points.shape[0], out.data_ptr(), self.hist_buf.data_ptr(),
                                       self.ws.data_ptr(), self.ws.numel(), self._st()))
        return out

    def hist(self, points, gbb, d_th):
        self._chk(self.L.fec_part_hist(self._p(points), points.shape[0], gbb.data_ptr(), _f32(d_th),
                                       self.hist_buf.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._st()))
        return self.hist_buf

    def plan(self, ghist, world):
        import torch
        plan = torch.empty(4 * world + 3, dtype=torch.int64, device=self.dev)
        self._chk(self.L.fec_part_plan(ghist.data_ptr(), world, plan.data_ptr(), self.ws.data_ptr(),
                                       self.ws.numel(), self._st()))
        return plan

    def count(self, points, gidx, gbb, d_th, plan, world):
        import torch
        counts = torch.empty(world, dtype=torch.int64, device=self.dev)
        self._chk(self.L.fec_part_pack(self._p(points), self._p(gidx), points.shape[0], gbb.data_ptr(), _f32(d_th),
                                       plan.data_ptr(), world, counts.data_ptr(), None, None, self.ws.data_ptr(),
                                       self.ws.numel(), self._st()))
        return counts

    def pack(self, points, gidx, gbb, d_th, plan, world, counts, total):
        import torch
        sp = torch.empty((max(total, 1), 3), dtype=torch.float32, device=self.dev)
        sg = torch.empty(max(total, 1), dtype=torch.int32, device=self.dev)
        if total:
            self._chk(self.L.fec_part_pack(self._p(points), self._p(gidx), points.shape[0], gbb.data_ptr(),
                                           _f32(d_th), plan.data_ptr(), world, counts.data_ptr(), sp.data_ptr(),
                                           sg.data_ptr(), self.ws.data_ptr(), self.ws.numel(), self._st()))
        return sp[:total], sg[:total]

    def order(self, rpts, rgidx, gbb, d_th, plan, world, rank):
        import torch
        k = rpts.shape[0]
        op = torch.empty((max(k, 1), 3), dtype=torch.float32, device=self.dev)
        og = torch.empty(max(k, 1), dtype=torch.int32, device=self.dev)
        c3 = torch.empty(3, dtype=torch.int64, device=self.dev)
        self._chk(self.L.fec_part_order(self._p(rpts), self._p(rgidx), k, gbb.data_ptr(), _f32(d_th),
                                        plan.data_ptr(), world, rank, c3.data_ptr(), self._p(op), self._p(og),
                                        self.ws.data_ptr(), self.ws.numel(), self._st()))
        return op[:k], og[:k], c3


def repartition(points, gidx, d_th: float, group=None, ops=None):
    """Mode B on this rank: `points` (float32 [m, 3]) / `gidx` (int32 [m]) is an arbitrary shard of
    the cloud; returns (Shard of this rank's slab in fec_slab_local's order, rec_cap).  Collective
    over `group`: one all-reduce of the bbox, one of the layer histogram, an all-to-all of the
    counts and one of the points / indices.  `ops` defaults to the device kernels (DevicePartOps);
    the split sizes of the all-to-all are the only device->host reads."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if ops is None:
        ops = DevicePartOps(points.device)
    bb = ops.bbox(points)
    if world > 1:
        dist.all_reduce(bb, op=dist.ReduceOp.MIN, group=group)
    hist = ops.hist(points, bb, d_th)
    if world > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    plan = ops.plan(hist, world)
    ph = plan.cpu().numpy()
    status = int(ph[4 * world + 2])
    if status:
        from . import FecError
        raise FecError(status, "Mode B partition: the global cloud cannot be cut (non-finite or extent)")
    rec_cap = int(ph[4 * world + 1])
    counts = ops.count(points, gidx, bb, d_th, plan, world)
    recv_counts = torch.empty_like(counts)
    if world > 1:
        dist.all_to_all_single(recv_counts, counts, group=group)
    else:
        recv_counts.copy_(counts)
    sc = counts.cpu().tolist()
    rc = recv_counts.cpu().tolist()
    sp, sg = ops.pack(points, gidx, bb, d_th, plan, world, counts, int(sum(sc)))
    rp = torch.empty((int(sum(rc)), 3), dtype=torch.float32, device=points.device)
    rg = torch.empty(int(sum(rc)), dtype=torch.int32, device=points.device)
    if world > 1:
        dist.all_to_all_single(rp, sp, rc, sc, group=group)
        dist.all_to_all_single(rg, sg, rc, sc, group=group)
    else:
        rp.copy_(sp)
        rg.copy_(sg)
    op, og, c3 = ops.order(rp, rg, bb, d_th, plan, world, rank)
    c = c3.cpu().tolist()
    return Shard(op, og, int(c[0] + c[1]), int(c[0])), rec_cap
