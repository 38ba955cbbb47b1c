#!/usr/bin/env python
"""FEC hot-path benchmark (driver contract: one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl fec|reference]

A step = one full pass of the hot path (validate+bbox, keys,
sort, gather, tables, neighbour scan + union, flatten, stats, relabel) over one resident
batch of synthetic points.  `value` = points clustered per second (Mpoints/s), CUDA-event
timed on the launching stream, max over ranks.  `e2e` = the same metric through the
host-buffer C-ABI call (fec_cluster_host: H2D points + D2H labels inside the timed region).
`roofline` = the dominant stage's algorithmic bytes / its event-timed duration vs the
measured HBM copy bandwidth.  `cpu_baseline` = the oracle (oracle/, 1 core) on a bounded
sample of the same workload.  `--impl reference` times that oracle instead (the
reference arm of this tier).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

WORKLOAD_TEXT = {
    "C1": "C1: 10k pts, 20 Gaussian blobs + 2k uniform noise, shuffled; d_th=0.5 m, min 10, max 1e6",
    "C2": "C2: one synthetic 64-beam LiDAR scan (~32k pts, ground removed); d_th=0.35 m, min 50, max 25k",
    "C3": "C3: 100-scan accumulated synthetic LiDAR map (~9M pts); d_th=0.2 m, min 50, max 1e6",
    "C4": "C4: 27M-pt accumulated synthetic LiDAR loop map (450 poses, 2,000 roadside objects); d_th=0.25 m, min 100, max 5e6",
    "C5": "C5: 100M uniform pts at mean degree 2.8 + 50 balls x 200k pts, shuffled; d_th=0.1 m, min 1, max 1e9",
}
# bounded oracle samples (prefixes in acquisition order for the LiDAR maps)
CPU_SAMPLE = {"C1": None, "C2": None, "C3": 4_000_000, "C4": 12_000_000, "C5": 8_000_000}
REF_STEP_SAMPLE = {"C1": None, "C2": None, "C3": 600_000, "C4": 1_200_000, "C5": 1_000_000}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C4", choices=sorted(synth.CONFIGS))
    ap.add_argument("--scale", type=float, default=1.0, help="shrink C3-C5 (tests only; not a bench value)")
    ap.add_argument("--impl", default="fec", choices=["fec", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--check", action="store_true", help="also verify the labels bit-exactly (untimed)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay one captured CUDA graph per step (auto: clouds of <= 2^20 points, whose "
                         "step is launch-bound); the call is fec_cluster_ws_async either way")
    ap.add_argument("--slab", action="store_true", help="use the slab (multi-GPU) path even at N=1 (testing)")
    ap.add_argument("--grid-mode", default="auto", choices=["auto", "hashed", "keysort", "countsort"],
                    help="testing: force a binning mode")
    ap.add_argument("--batch", type=int, default=0,
                    help="per-scan mode: cluster this many independent C2-recipe scans per step in one "
                         "fec_cluster_batch_ws call (SURVEY N1)")
    ap.add_argument("--ground", default="", choices=["", "G2", "G3"],
                    help="time the ground-removal pre-pass (SURVEY N2) on G2 (one scan) or G3 (100-scan map) "
                         "instead of clustering")
    ap.add_argument("--ap", action="store_true",
                    help="time the AP metric (SURVEY N3) on the paper's largest voxel-fill setting "
                         "(2,200 clusters x 500 points) against its ground truth")
    return ap.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.lines = []
        self.proc = None
        self.gpu = gpu_index

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-i", str(self.gpu), "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        time.sleep(0.15)
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for k, name in enumerate(names):
                if f[5 + k].lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


STAGE_KERNELS = {
    "a1_bbox_validate": "k_bbox (its last block plans the grid on the device), k_zero",
    "a2_bin_keys": "k_lkey + k_onesweep x passes (key path)",
    "a3_sort": "k_cmark / k_smark, k_cpop + k_tscan + k_cscan, k_dcount2 / k_sgather, k_cellred + k_celltscan + k_cellscan, "
               "k_dcomps",
    "a4_gather_init": "k_dscatter phase 0 (+ phase 1, enqueued after the dense links; node-tail clouds scatter "
                      "only the cells later kernels read), k_dinit, k_dparent",
    "a6a7_scan_union": "k_union_sparse(_local), k_dense_link x2 (the main-stream one also runs the "
                       "overflow fallback), k_dense_filter (with the node flattening), k_dense_overflow, k_dense_items",
    "a8_flatten": "k_flatten_if",
    "a9_stats": "k_tail_stats",
    "a10_relabel": "k_rootlab, k_relabel_in (node-tail clouds) / k_relabel_b1 (the bucket pass of large sparse-dominated clouds) + "
                   "k_relabel_b2c (a cluster per bucket) / k_relabel",
}


def roofline_stages(stages: dict) -> dict:
    """Stage times for the roofline: the two union stages form SURVEY's a6+a7 row."""
    out = {k: v for k, v in stages.items() if k not in ("a1_bbox_validate", "a6a7_union_sparse", "a6a7_union_dense")}
    out["a6a7_scan_union"] = stages.get("a6a7_union_sparse", 0.0) + stages.get("a6a7_union_dense", 0.0)
    return out


def algorithmic_bytes(stage: str, n: int, st: dict) -> float:
    """Bytes each stage must move: n points, C grid cells (bitmap index; hash
    mode: table slots), U occupied cells, nd dense cells, md points in dense cells, P key-sort
    passes (0 on the counting path)."""
    C = float(np.prod(st["dims"])) if st["dense_table"] == 1 else 4.0 * n
    U = float(max(st.get("cells", 0), 0))  # occupied cells
    nd = float(max(st.get("dense_cells", 0), 0))
    md = float(max(st.get("dense_points", 0), 0))
    P = float(max(st.get("radix_passes", 0), 0))
    ns = n - md                             # points of sparse cells
    key = P > 0
    model = {
        "a1_bbox_validate": 12.0 * n,
        # key path: read xyz, write key + index (+ histograms), then per pass read + write 8 B
        "a2_bin_keys": (12.0 * n + 8.0 * n + 16.0 * n * P) if key else 0.0,
        # bitmap (C/8 B, ~9 touches), cell lists (28 B/cell), xyz reads, counts + fine masks,
        # scan, dense records + components (~180 B/dense cell); key path: keys instead of xyz
        "a3_sort": (8.0 * n + 1.125 * C + 44.0 * U + 24.0 * U + 180.0 * nd + 12.0 * n + 16.0 * n) if key else
                   (24.0 * n + 1.125 * C + 44.0 * U + 24.0 * U + 180.0 * nd),
        # count path: xyz -> float4 scatter, float4 -> parent, idx (+ root accumulators)
        "a4_gather_init": (8.0 * md) if key else (12.0 * n + 16.0 * n + 16.0 * n + 8.0 * n + 8.0 * ns),
        "a5_tables": 0.0,
        # SURVEY §8(d) B_model for the neighbour scan + union-find (a6+a7): 28 B per point
        # (float4 read 16 + parent init / hook 12), over the two union stages together
        "a6a7_scan_union": 28.0 * n,
        "a8_flatten": 8.0 * n if 4 * U > n else 0.0,          # separate flatten (sparse-dominated only)
        # node tail (few sparse cells): sparse points + 8 node slots per dense cell
        "a9_stats": (12.0 * ns + 64.0 * nd) if 4 * U <= n else 12.0 * n,
        "a10_relabel": 12.0 * n,                              # parent + index -> label
    }
    return model[stage]


def dist_setup(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # testing aids (not used by the driver): FEC_DIST_BACKEND=gloo and FEC_FORCE_DEVICE=0 let
    # several ranks share one GPU to exercise the multi-rank code path end to end
    local = int(os.environ.get("FEC_FORCE_DEVICE", local))
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("FEC_DIST_BACKEND", "nccl") if args.impl == "fec" else "gloo"
        if args.impl == "fec":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    elif args.impl == "fec":
        torch.cuda.set_device(local)
    return rank, world, local


def make_workload(name: str, scale: float, limit: int | None = None):
    if limit is not None and name in ("C3", "C4"):
        # acquisition-order prefix: whole poses, generated without building the full map
        if name == "C4":
            k = 1
            while True:
                pts = synth.c4_loop(3, pose_range=(0, k))
                if pts.shape[0] >= limit or k >= 450:
                    break
                k = max(k + 1, int(k * limit / max(pts.shape[0], 1)))
            return pts[:limit], f"first {min(limit, pts.shape[0])} points (first {k} poses) of C4"
        w = synth.make_config(name, scale=min(1.0, scale))
        return w.points[:limit], f"first {limit} points of C3"
    w = synth.make_config(name, scale=scale)
    if limit is not None and w.n > limit:
        return w.points[:limit], f"first {limit} points of {name} (shuffled order = uniform subsample)"
    return w.points, f"all {w.n} points of {name}"


def run_reference(args, rank, world):
    import oracle
    if rank != 0:
        return
    d, mn, mx = synth.CONFIGS[args.config]
    limit = REF_STEP_SAMPLE[args.config]
    pts, desc = make_workload(args.config, args.scale, limit)
    n = pts.shape[0]
    times = []
    with pinned_core():
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.fec(pts, d, mn, mx)
            dt = time.perf_counter() - t0
            if k >= args.warmup:
                times.append(dt)
    mean = float(np.mean(times))
    value = n / mean / 1e6
    line = {
        "impl": "reference", "metric": "Mpoints/s clustered", "value": value, "unit": "Mpoints/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": WORKLOAD_TEXT[args.config], "n_points_per_step": n, "sample": desc},
        "cpu_baseline": {"value": value, "unit": "Mpoints/s", "cores": 1, "kind": "oracle",
                         "sample": desc + "; pinned to core 0", **host_cpu()},
        "e2e": {"value": value, "unit": "Mpoints/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def host_cpu() -> dict:
    """The GPU box's host CPU (SURVEY §8(d) "Oracle timing": model, nproc, the pinned core)."""
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


class pinned_core:
    """Runs the enclosed code on core 0 only (taskset -c 0 equivalent), then restores."""

    def __enter__(self):
        self.prev = None
        try:
            self.prev = os.sched_getaffinity(0)
            os.sched_setaffinity(0, {0})
        except (AttributeError, OSError):
            self.prev = None
        return self

    def __exit__(self, *a):
        if self.prev is not None:
            os.sched_setaffinity(0, self.prev)


def cpu_baseline(name: str, scale: float):
    import oracle
    d, mn, mx = synth.CONFIGS[name]
    pts, desc = make_workload(name, scale, CPU_SAMPLE[name])
    with pinned_core():
        t0 = time.perf_counter()
        oracle.fec(pts, d, mn, mx)
        dt = time.perf_counter() - t0
    return {"value": pts.shape[0] / dt / 1e6, "unit": "Mpoints/s", "cores": 1, "kind": "oracle",
            "sample": f"{desc}; {dt:.1f} s single-threaded, pinned to core 0", **host_cpu()}


def run_slab(args, rank: int, world: int, local: int):
    """N > 1: the cloud is sharded into spatial slabs (+ one-cell halo) before the timed
    region (north_star: "sharded across the 8xB200 box into spatial slabs"); a step is
    fec_slab_local -> NCCL all-gather of boundary records -> fec_slab_merge on every rank.
    Total work is the fixed workload, so scaling is strong."""
    import torch
    import torch.distributed as tdist
    import paper_2208_07678_b200 as fec
    from paper_2208_07678_b200 import dist as fdist

    multi = world > 1

    def barrier():
        if multi:
            tdist.barrier()

    def allreduce(t, op=tdist.ReduceOp.SUM):
        if multi:
            tdist.all_reduce(t, op=op)
        return t

    fec.lib()
    d_th, mn, mx = synth.CONFIGS[args.config]
    w = synth.make_config(args.config, scale=args.scale)
    n_total = w.n
    plan = fdist.plan_slabs(w.points, d_th, world)  # identical on every rank
    sh = fdist.shard(w.points, plan, rank)
    dev = torch.device("cuda", local)
    x = torch.from_numpy(sh.points).to(dev)
    g = torch.from_numpy(sh.gidx).to(dev)
    runner = fdist.SlabRunner(x, g, sh.n_owned, sh.n_first, plan.rec_cap, d_th, mn, mx, world, rank)
    stream = torch.cuda.current_stream(dev)
    fec.set_instrumentation(True)
    runner.step()
    torch.cuda.synchronize()
    st = fec.stats()
    fec.set_instrumentation(False)
    check = None
    if args.check:
        import oracle
        parts = [None] * world
        mine = (sh.gidx[:sh.n_owned], runner.labels.cpu().numpy())
        if multi:
            tdist.all_gather_object(parts, mine)
        else:
            parts = [mine]
        if rank == 0:
            full = np.full(n_total, -7, np.int32)
            for gi, lab in parts:
                full[gi] = lab
            check = bool(np.array_equal(full, oracle.fec(w.points, d_th, mn, mx)))
    for _ in range(args.warmup):
        runner.step()
    torch.cuda.synchronize()
    barrier()
    stage_sum: dict[str, float] = {}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            runner.step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms_local = e0.elapsed_time(e1) / args.steps
    # per-stage times in a second pass (the stage events split the stream)
    fec.set_timing(True)
    for _ in range(args.steps):
        runner.step()
        for k, v in fec.stage_times().items():
            stage_sum[k] = stage_sum.get(k, 0.0) + v
    fec.set_timing(False)
    torch.cuda.synchronize()
    barrier()
    t = torch.tensor([ms_local], device=dev)
    allreduce(t, op=tdist.ReduceOp.MAX)
    ms = float(t.item())
    value = n_total / (ms * 1e-3) / 1e6

    # e2e: this rank's slab from pinned host memory, labels back to host, every step
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(sh.points).pin_memory()
        hg = torch.from_numpy(sh.gidx).pin_memory()
        hl = torch.empty(sh.n_owned, dtype=torch.int32).pin_memory()

        def host_step():
            runner.points.copy_(hp, non_blocking=True)
            runner.gidx.copy_(hg, non_blocking=True)
            lab = runner.step()
            hl.copy_(lab, non_blocking=True)
            stream.synchronize()

        for _ in range(max(1, args.warmup // 2)):
            host_step()
        barrier()
        ksteps = max(3, args.steps // 2)
        e0.record(stream)
        for _ in range(ksteps):
            host_step()
        e1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / ksteps], device=dev)
        allreduce(t, op=tdist.ReduceOp.MAX)
        ems = float(t.item())
        nb = torch.tensor([16 * sh.points.shape[0], 4 * sh.n_owned], device=dev, dtype=torch.int64)
        allreduce(nb)  # bytes copied by all ranks together
        e2e = {"value": n_total / (ems * 1e-3) / 1e6, "unit": "Mpoints/s",
               "h2d_bytes_per_step": int(nb[0].item()), "d2h_bytes_per_step": int(nb[1].item()),
               "ms_per_step": ems}

    n_local = sh.points.shape[0]
    stages = {k: v / args.steps for k, v in stage_sum.items()}
    rs = roofline_stages(stages)
    dom = max(rs, key=lambda k: rs[k])
    peak, peak_src = load_peaks()
    ab = algorithmic_bytes(dom, n_local, st)
    ach = ab / (rs[dom] * 1e-3) / 1e9
    roofline = {"bound": "hbm", "kernel": dom, "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": None, "peak_source": peak_src, "algorithmic_bytes": ab, "rank": rank}
    launches = torch.tensor([st["launches"] + 5], device=dev)  # + merge kernels
    allreduce(launches, op=tdist.ReduceOp.MAX)
    if rank == 0:
        line = {
            "metric": "Mpoints/s clustered", "value": value, "unit": "Mpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[args.config] + ("" if args.scale == 1.0 else f" (scale {args.scale})"),
                       "n_points": n_total, "d_th": d_th, "min_size": mn, "max_size": mx,
                       "parallelism": f"slab{world} (axis {'xyz'[plan.axis]}, one-cell halo, NCCL all-gather "
                                      f"of boundary records)",
                       "slab_points": [int(v) for v in plan.n_owned], "halo_points": [int(v) for v in plan.n_halo],
                       "rec_cap": plan.rec_cap,
                       "l2": "no flush: per-rank inputs and working set exceed the 126 MB L2"
                             if 12 * n_local > 126e6 else "per-rank input below L2 size; working set "
                             f"({fec.slab_workspace_bytes(n_local, world, plan.rec_cap) / 1e9:.2f} GB) exceeds it"},
            "e2e": e2e,
            "roofline": roofline,
            "cpu_baseline": None,
            "gpu_launches": int(launches.item()) * args.steps,
            "clocks": clk.summary(),
            "stages_ms_rank0": stages,
        }
        if check is not None:
            line["parity_bit_exact"] = check
        print(json.dumps(line), flush=True)
    if multi:
        tdist.destroy_process_group()


def run_batch(args, local: int):
    """Per-scan mode (the paper's Table 4 setting): B independent single scans (C2 recipe,
    seeds 1000..) per step, one batched call; the same scans through B separate calls are
    timed beside it."""
    import torch
    import paper_2208_07678_b200 as fec
    fec.lib()
    d_th, mn, mx = synth.CONFIGS["C2"]
    scans = [synth.lidar_scan(1000 + k) for k in range(args.batch)]
    offs = np.concatenate([[0], np.cumsum([len(c) for c in scans])]).astype(np.int64)
    pts = np.concatenate(scans)
    n = pts.shape[0]
    dev = torch.device("cuda", local)
    x = torch.from_numpy(pts).to(dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    ws = torch.empty(fec.batch_workspace_bytes(n, len(scans)), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    check = None
    if args.check:
        import oracle
        fec.cluster_batch(x, offs, d_th, mn, mx, out=out, workspace=ws)
        got = out.cpu().numpy()
        check = all(np.array_equal(got[offs[k]:offs[k + 1]], oracle.fec(scans[k], d_th, mn, mx))
                    for k in range(len(scans)))
    for _ in range(args.warmup):
        fec.cluster_batch(x, offs, d_th, mn, mx, out=out, workspace=ws)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            fec.cluster_batch(x, offs, d_th, mn, mx, out=out, workspace=ws)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # the same scans, one call each (workspace reused)
    wss = torch.empty(fec.workspace_bytes(max(len(c) for c in scans)), dtype=torch.uint8, device=dev)
    xs = [x[offs[k]:offs[k + 1]] for k in range(len(scans))]
    e0.record(stream)
    for _ in range(max(1, args.steps // 3)):
        for k in range(len(scans)):
            fec.cluster(xs[k], d_th, mn, mx, out=out[offs[k]:offs[k + 1]], workspace=wss, check=False)
    e1.record(stream)
    torch.cuda.synchronize()
    ms_seq = e0.elapsed_time(e1) / max(1, args.steps // 3)
    line = {
        "metric": "Mpoints/s clustered", "value": n / (ms * 1e-3) / 1e6, "unit": "Mpoints/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"per-scan mode: {len(scans)} independent C2-recipe scans (seeds 1000..) in one "
                               f"fec_cluster_batch_ws call; d_th=0.35 m, min 50, max 25k",
                   "n_points": int(n), "scans": len(scans), "parallelism": "single",
                   "l2": "inputs below L2 size (latency-bound)" if 12 * n < 126e6 else "inputs exceed L2"},
        "sequential_calls_ms_per_step": ms_seq,
        "sequential_calls_mpts_s": n / (ms_seq * 1e-3) / 1e6,
        "clocks": clk.summary(),
    }
    if check is not None:
        line["parity_bit_exact"] = bool(check)
    print(json.dumps(line), flush=True)


def fp32_alu_peak_tflops(sm_mhz=None) -> float:
    """Non-tensor fp32 FMA peak: 148 SMs x 128 FP32 lanes x 2 flops x clock."""
    mhz = sm_mhz or 1965.0
    return 148 * 128 * 2 * mhz * 1e6 / 1e12


def run_ground(args, local: int):
    """Ground removal (RANSAC plane fit) on G2/G3: H = 100 hypotheses, every
    point tested against every plane (the dominant kernel k_g_count: 3 fused multiply-adds per
    test), then the best plane's survivors compacted.  ALU roofline of k_g_count."""
    import math
    import torch
    import paper_2208_07678_b200 as fec
    fec.lib()
    pts, tri, thr, tilt = synth.make_ground_config(args.ground)
    n, H = pts.shape[0], tri.shape[0]
    ct = math.cos(math.radians(tilt))
    dev = torch.device("cuda", local)
    x = torch.from_numpy(pts).to(dev)
    t = torch.from_numpy(tri).to(dev)
    out = (torch.empty((n, 3), dtype=torch.float32, device=dev), torch.empty(n, dtype=torch.int32, device=dev),
           torch.empty(fec.GROUND_RESULT_BYTES, dtype=torch.uint8, device=dev))
    ws = torch.empty(fec.ground_workspace_bytes(n, H), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        return fec.remove_ground(x, t, thr, cos_max_tilt=ct, out=out, workspace=ws)

    step()
    torch.cuda.synchronize()
    info = fec.ground_result(out[2])
    check = None
    if args.check:
        from oracle import ground as og
        w = og.ransac_ground(pts, tri, thr, ct, (n + 9) // 10)
        check = bool(w.best == info["best"] and np.array_equal(out[1][:info["n_keep"]].cpu().numpy(), w.keep_idx))
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    fec.set_timing(True)   # events around k_g_count inside each call (same stream)
    kms = 0.0
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
            kms += fec.ground_count_ms()
        e1.record(stream)
        torch.cuda.synchronize()
    fec.set_timing(False)
    kms /= args.steps
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.summary()
    # e2e: pinned host points + triplets in, result record + survivor indices out
    e2e = None
    if not args.no_e2e:
        hp = torch.from_numpy(pts).pin_memory()
        ht = torch.from_numpy(tri).pin_memory()
        hk = torch.empty(n, dtype=torch.int32).pin_memory()
        hr = torch.empty(fec.GROUND_RESULT_BYTES, dtype=torch.uint8).pin_memory()

        def host_step():
            x.copy_(hp, non_blocking=True)
            t.copy_(ht, non_blocking=True)
            fec.remove_ground(x, t, thr, cos_max_tilt=ct, out=out, workspace=ws)
            hr.copy_(out[2], non_blocking=True)
            hk.copy_(out[1], non_blocking=True)

        for _ in range(2):
            host_step()
        torch.cuda.synchronize()
        k = max(3, args.steps // 2)
        e0.record(stream)
        for _ in range(k):
            host_step()
        e1.record(stream)
        torch.cuda.synchronize()
        ems = e0.elapsed_time(e1) / k
        e2e = {"value": n / (ems * 1e-3) / 1e6, "unit": "Mpoints/s", "h2d_bytes_per_step": 12 * n + 12 * H,
               "d2h_bytes_per_step": 4 * n + fec.GROUND_RESULT_BYTES, "ms_per_step": ems}
    tests = float(n) * H
    flops = 6.0 * tests  # 3 FMA per point-plane test
    peak = fp32_alu_peak_tflops(clocks.get("sm_max_mhz"))
    cpu = None
    if not args.no_cpu_baseline:
        from oracle import ground as og
        hs = 4 if args.ground == "G3" else H
        t0 = time.perf_counter()
        og.counts(pts, tri[:hs], thr, ct)
        dt = time.perf_counter() - t0
        cpu = {"value": n * (hs / H) / dt / 1e6, "unit": "Mpoints/s", "cores": 1, "kind": "oracle",
               "sample": f"oracle inlier counting of {hs} of the {H} hypotheses over all {n} points "
                         f"(scaled to the full {H}-hypothesis step)"}
    line = {
        "metric": "Mpoints/s ground-removed", "value": n / (ms * 1e-3) / 1e6, "unit": "Mpoints/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.ground}: RANSAC plane-fit ground removal (SURVEY N2), {H} hypotheses, "
                               f"threshold {thr} m, max tilt {tilt} deg, ground kept in the LiDAR recipe, tilted 2 deg",
                   "n_points": int(n), "hypotheses": int(H), "ground_points": int(info["n_inliers"]),
                   "parallelism": "single",
                   "l2": "inputs exceed L2" if 12 * n > 126e6 else "inputs below L2 size"},
        "e2e": e2e,
        "roofline": {"bound": "alu", "kernel": "k_g_count", "achieved": flops / (kms * 1e-3) / 1e12,
                     "peak": peak, "unit": "TFLOP/s", "frac": flops / (kms * 1e-3) / 1e12 / peak, "traffic": None,
                     "kernel_ms": kms, "algorithmic_flops": flops,
                     "peak_source": "derived: 148 SMs x 128 fp32 lanes x 2 x max SM clock (DESIGN.md §8c)"},
        "cpu_baseline": cpu,
        "gpu_launches": 7 * args.steps,  # planes, count, best, flags, scan, compact, refine
        "clocks": clocks,
    }
    if check is not None:
        line["parity_bit_exact"] = check
    print(json.dumps(line), flush=True)


def run_ap(args, local: int):
    """AP (Eq. 2, 0.75 IoU) of the clustering path's labels against the voxel generator's ground
    truth, P:L281 setting at its largest size (Fig. 4: 2,200 clusters, density 500)."""
    import torch
    import paper_2208_07678_b200 as fec
    fec.lib()
    pts, gt, d = synth.voxel_clusters(2200, 500, shift_sigma=0.0, seed=0)
    n = pts.shape[0]
    dev = torch.device("cuda", local)
    x = torch.from_numpy(pts).to(dev)
    g = torch.from_numpy(gt).to(dev)
    lab = fec.cluster(x, d)
    ws = torch.empty(fec.ap_workspace_bytes(n), dtype=torch.uint8, device=dev)
    res = torch.empty(fec.AP_RESULT_BYTES, dtype=torch.uint8, device=dev)
    r = fec.average_precision(lab, g, 0.75, workspace=ws, result=res)
    check = None
    if args.check:
        from oracle.metrics import average_precision as ap_or
        w = ap_or(lab.cpu().numpy(), gt)
        check = bool(w["tp"] == r["tp"] and w["fp"] == r["fp"])
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        fec.average_precision(lab, g, 0.75, workspace=ws, result=res, read=False)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            fec.average_precision(lab, g, 0.75, workspace=ws, result=res, read=False)
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    # e2e: host labels in, result record out
    hl = lab.cpu().pin_memory()
    hg = torch.from_numpy(gt).pin_memory()
    hr = torch.empty(fec.AP_RESULT_BYTES, dtype=torch.uint8).pin_memory()
    lab2 = torch.empty_like(lab)
    g2 = torch.empty_like(g)
    k = max(3, args.steps // 2)
    e0.record(stream)
    for _ in range(k):
        lab2.copy_(hl, non_blocking=True)
        g2.copy_(hg, non_blocking=True)
        fec.average_precision(lab2, g2, 0.75, workspace=ws, result=res, read=False)
        hr.copy_(res, non_blocking=True)
    e1.record(stream)
    torch.cuda.synchronize()
    ems = e0.elapsed_time(e1) / k
    bits = 2 * int(np.ceil(np.log2(n + 2)))
    passes = 2 * ((bits + 7) // 8)
    model = 8.0 * n + passes * 28.0 * n + 40.0 * n  # labels in; 2 sorts x passes x (key+val r/w + hist); runs/keys
    peak, src = load_peaks()
    t0 = time.perf_counter()
    from oracle.metrics import average_precision as ap_or
    ap_or(lab.cpu().numpy(), gt)
    cpu_s = time.perf_counter() - t0
    line = {
        "metric": "Mpoints/s scored (AP, Eq. 2)", "value": n / (ms * 1e-3) / 1e6, "unit": "Mpoints/s", "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": {"workload": "AP of fec_cluster's labels vs ground truth, voxel-fill setting (P:L281) with "
                               "2,200 clusters x 500 points, threshold 0.75",
                   "n_points": int(n), "tp": r["tp"], "fp": r["fp"], "ap": r["ap"], "parallelism": "single",
                   "l2": "inputs below L2 size"},
        "e2e": {"value": n / (ems * 1e-3) / 1e6, "unit": "Mpoints/s", "h2d_bytes_per_step": 8 * n,
                "d2h_bytes_per_step": fec.AP_RESULT_BYTES, "ms_per_step": ems},
        "roofline": {"bound": "hbm", "kernel": "whole step (radix sorts of the pair histogram dominate)",
                     "achieved": model / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                     "frac": model / (ms * 1e-3) / 1e9 / peak, "traffic": None, "peak_source": src,
                     "algorithmic_bytes": model},
        "cpu_baseline": {"value": n / cpu_s / 1e6, "unit": "Mpoints/s", "cores": 1, "kind": "oracle",
                         "sample": f"oracle AP over all {n} points"},
        "gpu_launches": (10 + 3 * passes) * args.steps,  # 2 sorts x passes x (hist, scan, scatter) + 10 "clocks": clk.summary(),
    }
    if check is not None:
        line["parity_bit_exact"] = check
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if args.ap and world == 1:
        run_ap(args, local)
        return
    if args.ground and world == 1:
        run_ground(args, local)
        return
    if args.batch > 1 and world == 1:
        run_batch(args, local)
        return
    if world > 1 or args.slab:
        run_slab(args, rank, world, local)
        return
    import torch
    import paper_2208_07678_b200 as fec

    fec.lib()
    fec.set_grid_mode({"auto": 0, "hashed": 1, "keysort": 2, "countsort": 3}[args.grid_mode])
    d_th, mn, mx = synth.CONFIGS[args.config]
    w = synth.make_config(args.config, scale=args.scale)
    n = w.n
    dev = torch.device("cuda", local)
    x = torch.from_numpy(w.points).to(dev)
    out = torch.empty(n, dtype=torch.int32, device=dev)
    ws = torch.empty(fec.workspace_bytes(n), dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    # one instrumented, untimed call: sizes for the byte model + launch count
    fec.set_instrumentation(True)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    fec.cluster(x, d_th, mn, mx, out=out, workspace=ws, status=status)
    torch.cuda.synchronize()
    st = fec.stats()
    fec.set_instrumentation(False)
    check = None
    if args.check:
        import oracle
        check = bool(np.array_equal(out.cpu().numpy(), oracle.fec(w.points, d_th, mn, mx)))

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def call():
        fec.cluster(x, d_th, mn, mx, out=out, workspace=ws, status=status, check=False)

    use_graph = args.graph == "on" or (args.graph == "auto" and n <= (1 << 20))
    step = call
    if use_graph:
        # the whole call has no host round trip (the grid is planned on the device), so one
        # captured graph replays the complete step: launch-bound small clouds are timed
        # without the host's per-launch cost
        graph = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream(dev)
        cs.wait_stream(stream)
        with torch.cuda.stream(cs):
            call()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=cs):
            call()
        torch.cuda.synchronize()
        step = graph.replay
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    barrier()

    stage_sum: dict[str, float] = {}
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1) / args.steps
    fec.raise_status(status)  # the device status of the timed calls (read after the timed region)
    digest = full_size_digest(args, w, out) if rank == 0 else None
    # per-stage times (library events at the stage boundaries) in a second pass of the same
    # steps: the events split the stream, so they are kept out of the timed loop
    fec.set_timing(True)
    for _ in range(args.steps):
        fec.cluster(x, d_th, mn, mx, out=out, workspace=ws, status=status, check=False)
        for k, v in fec.stage_times().items():
            stage_sum[k] = stage_sum.get(k, 0.0) + v
    fec.set_timing(False)
    torch.cuda.synchronize()
    # SURVEY 8(d) also asks for the median and min of the timed runs: K more steps, each
    # bracketed by its own events (a separate pass, so the timed loop above stays unsplit)
    per_step = []
    for _ in range(args.steps):
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        step()
        a1.record(stream)
        a1.synchronize()
        per_step.append(a0.elapsed_time(a1))
    per_step.sort()
    step_stats = {"median_ms": per_step[len(per_step) // 2], "min_ms": per_step[0], "max_ms": per_step[-1],
                  "runs": len(per_step), "note": "separate pass after the timed loop, one event pair per step"}
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    total_points = n * world
    value = total_points / (ms * 1e-3) / 1e6

    # ---- e2e through the host-buffer C-ABI call ---------------------------------------------
    e2e = None
    if not args.no_e2e:
        # the public host-buffer API, pipelined two deep (fec_cluster_host_async on two
        # streams, each with its own workspace and pinned buffers): every step copies its
        # points in and its labels out inside the timed region; consecutive steps overlap one
        # step's device->host copy with the next step's host->device copy
        hp = [torch.from_numpy(w.points).pin_memory() for _ in range(2)]
        hl = [torch.empty(n, dtype=torch.int32).pin_memory() for _ in range(2)]
        wsh = [torch.empty(fec.workspace_bytes_host(n), dtype=torch.uint8, device=dev) for _ in range(2)]
        sts = [torch.cuda.Stream(dev) for _ in range(2)]
        for k in range(max(2, args.warmup // 2)):
            fec.cluster_host(hp[k % 2], d_th, mn, mx, out=hl[k % 2], workspace=wsh[k % 2], stream=sts[k % 2],
                             sync=False)
        torch.cuda.synchronize()
        barrier()
        ksteps = max(4, args.steps // 2)
        ea = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e0.record(sts[0])
        sts[1].wait_event(e0)
        for k in range(ksteps):
            fec.cluster_host(hp[k % 2], d_th, mn, mx, out=hl[k % 2], workspace=wsh[k % 2], stream=sts[k % 2],
                             sync=False)
        for j in range(2):
            ea[j].record(sts[j])
        torch.cuda.synchronize()
        ems = max(e0.elapsed_time(ea[0]), e0.elapsed_time(ea[1])) / ksteps
        if check is not None and not np.array_equal(hl[(ksteps - 1) % 2].numpy(), out.cpu().numpy()):
            check = False
        if world > 1:
            t = torch.tensor([ems], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": total_points / (ems * 1e-3) / 1e6, "unit": "Mpoints/s",
               "h2d_bytes_per_step": 12 * n, "d2h_bytes_per_step": 4 * n, "ms_per_step": ems,
               "api": "fec_cluster_host_async, 2 streams (steps overlap copy directions)"}
        del wsh

    # ---- roofline of the dominant stage -------------------------------------------------------
    stages = {k: v / args.steps for k, v in stage_sum.items()}
    rs = roofline_stages(stages)
    dom = max(rs, key=lambda k: rs[k])
    peak, peak_src = load_peaks()
    ach = algorithmic_bytes(dom, n, st) / (rs[dom] * 1e-3) / 1e9
    tinfo = {}
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        try:
            tinfo = json.load(open(tfile)).get(args.config, {})
        except Exception:
            tinfo = {}

    def traffic_of(stage):
        e = tinfo.get(stage)
        return e.get("dram_bytes") if isinstance(e, dict) else None

    roofline = {"bound": "hbm", "kernel": dom, "kernels": STAGE_KERNELS.get(dom, dom), "achieved": ach,
                "peak": peak, "unit": "GB/s", "frac": ach / peak, "traffic": traffic_of(dom), "peak_source": peak_src,
                "algorithmic_bytes": algorithmic_bytes(dom, n, st), "stage_ms": rs[dom],
                "traffic_source": tinfo.get("source")}
    # the north star's target stage (neighbour scan + union-find, 28 B/pt), reported
    # whether or not it dominates; its dense-dense links run on a side stream concurrently with
    # the scatter, so its main-stream stage time excludes them -- the ncu sum of its kernels
    # (serialised, cold cache) is given beside it
    a67 = rs.get("a6a7_scan_union", 0.0)
    a67_bytes = algorithmic_bytes("a6a7_scan_union", n, st)
    e67 = tinfo.get("a6a7_scan_union") if isinstance(tinfo.get("a6a7_scan_union"), dict) else {}
    roofline_a6a7 = {"bound": "hbm", "kernel": "a6a7_scan_union", "kernels": STAGE_KERNELS["a6a7_scan_union"],
                     "achieved": a67_bytes / (a67 * 1e-3) / 1e9 if a67 > 0 else None, "peak": peak, "unit": "GB/s",
                     "frac": a67_bytes / (a67 * 1e-3) / 1e9 / peak if a67 > 0 else None,
                     "traffic": e67.get("dram_bytes"), "stage_ms": a67,
                     "ncu_kernels_us_incl_side_stream": e67.get("ncu_us"),
                     "algorithmic_bytes": a67_bytes}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args.config, args.scale)

    if rank == 0:
        line = {
            "metric": "Mpoints/s clustered", "value": value, "unit": "Mpoints/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD_TEXT[args.config] + ("" if args.scale == 1.0 else f" (scale {args.scale})"),
                       "n_points": n, "d_th": d_th, "min_size": mn, "max_size": mx,
                       "parallelism": "single",
                       "timing": ("one captured CUDA graph of the call replayed per step" if use_graph else
                                  "one fec_cluster_ws_async call per step, enqueued from Python"),
                       "l2": f"no flush: inputs ({12 * n / 1e6:.0f} MB) and working set "
                             f"({fec.workspace_bytes(n) / 1e9:.1f} GB) exceed the 126 MB L2"
                             if 12 * n > 126e6 else "small input: L2-resident (latency-bound)",
                       "cells": st["cells"], "groups": st["groups"], "components": st["components"],
                       "pair_tests": st["pair_tests"], "group_pairs": st["group_pairs"],
                       "dense_cells": st["dense_cells"], "dense_points": st["dense_points"],
                       "dense_tests": st["dense_tests"],
                       "radix_passes": st["radix_passes"], "dense_table": st["dense_table"],
                       "grid_dims": st["dims"]},
            "e2e": e2e,
            "roofline": roofline,
            "roofline_a6a7": roofline_a6a7,
            "cpu_baseline": cpu,
            "gpu_launches": st["launches"] * args.steps,
            "clocks": clk.summary(),
            "stages_ms": stages,
            "step_ms": step_stats,
        }
        if check is not None:
            line["parity_bit_exact"] = check
        if digest is not None:
            line["parity_digest"] = digest
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def full_size_digest(args, w, out):
    """The last timed step's labels against the ORACLE's stored full-size digest
    (tests/golden/full_size.json, written by tools/make_full_size_digests.py from synth/ and
    oracle/ only), after the timed region: the bench line itself says whether the input was
    the stored cloud and whether the measured step produced the oracle's labels."""
    if args.scale != 1.0 or args.grid_mode != "auto":
        return None
    import hashlib
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden", "full_size.json")
    try:
        ref = json.load(open(path))["configs"][args.config]
    except (OSError, KeyError, ValueError):
        return None
    in_sha = synth.sha256_f32(w.points)
    lab = np.ascontiguousarray(out.cpu().numpy(), dtype="<i4")
    return {"input_sha256": in_sha, "input_matches_golden": in_sha == ref["input_sha256"],
            "labels_match_oracle_digest": hashlib.sha256(lab.tobytes()).hexdigest() == ref["labels_sha256"],
            "source": "tests/golden/full_size.json (oracle labels, sha256)"}


if __name__ == "__main__":
    main()
