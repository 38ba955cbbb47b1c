"""Python binding of the FEC B200 library (argument marshalling only).

Every step of the path runs in libfec.so's sm_100a kernels behind the C ABI declared in
include/fec.h; this module only converts tensors to pointers, takes device memory for the
workspace from PyTorch's caching allocator and passes PyTorch's current CUDA stream.
There is no CPU fallback: if libfec.so is missing or no CUDA device is present, calls
raise.

    labels = cluster(points_cuda_f32_nx3, d_th, min_size, max_size)   # int32 [n], device
    labels = cluster_host(points_np, d_th, min_size, max_size)        # host in, host out
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

__all__ = ["average_precision", "ap_workspace_bytes", "remove_ground", "expand_labels", "cluster_nonground", "ground_result", "ground_workspace_bytes",
           "cluster", "cluster_async", "raise_status", "cluster_host", "cluster_batch", "batch_workspace_bytes", "slab_local", "slab_merge", "slab_record_words",
           "slab_workspace_bytes", "SlabState", "workspace_bytes", "workspace_bytes_host", "stats",
           "set_instrumentation", "set_timing", "stage_times", "FecError", "lib", "LIB_PATH", "debug_pred", "EXPORTS"]

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libfec.so")

OK, ERR_INVALID_ARGUMENT, ERR_NONFINITE, ERR_GRID_RANGE, ERR_OUT_OF_MEMORY, ERR_CUDA = 0, -1, -2, -3, -4, -5

# every symbol include/fec.h, include/fec_ground.h and include/fec_metrics.h declare
EXPORTS = ("fec_workspace_bytes", "fec_cluster_ws", "fec_cluster", "fec_cluster_async", "fec_cluster_ws_async",
           "fec_debug_alloc_extra", "fec_max_points", "fec_workspace_bytes_host",
           "fec_cluster_host", "fec_cluster_host_async", "fec_get_stats", "fec_set_instrumentation", "fec_status_string",
           "fec_last_error", "fec_version", "fec_debug_pred", "fec_set_timing",
           "fec_get_stage_times", "fec_stage_name", "fec_set_grid_mode", "fec_slab_record_words",
           "fec_slab_workspace_bytes", "fec_slab_local", "fec_slab_merge", "fec_set_item_cap",
           "fec_debug_subcell_tables", "fec_debug_subcell_dilate", "fec_debug_subcell_components",
           "fec_batch_workspace_bytes", "fec_cluster_batch_ws",
           "fec_part_workspace_bytes", "fec_part_max_layers", "fec_part_bbox", "fec_part_hist", "fec_part_plan",
           "fec_part_pack", "fec_part_order",
           # include/fec_ground.h
           "fec_ground_workspace_bytes", "fec_ground_remove", "fec_ground_expand_labels", "fec_ground_count_ms",
           # include/fec_metrics.h
           "fec_ap_workspace_bytes", "fec_average_precision")


class FecStats(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int64), ("cells", ctypes.c_int64), ("groups", ctypes.c_int64),
                ("components", ctypes.c_int64), ("pair_tests", ctypes.c_int64),
                ("group_pairs", ctypes.c_int64), ("dense_cells", ctypes.c_int64),
                ("dense_points", ctypes.c_int64), ("dense_tests", ctypes.c_int64),
                ("key_bits", ctypes.c_int64),
                ("radix_passes", ctypes.c_int32), ("dense_table", ctypes.c_int32),
                ("dims", ctypes.c_int32 * 3), ("launches", ctypes.c_int32), ("binning", ctypes.c_int32)]


class SlabState(ctypes.Structure):
    """Opaque host-side state carried from slab_local to slab_merge (fec_slab_state_t)."""
    _fields_ = [("opaque", ctypes.c_int64 * 8)]


class GroundResult(ctypes.Structure):
    """fec_ground_result_t (include/fec_ground.h)."""
    _fields_ = [("best", ctypes.c_int32), ("n_valid", ctypes.c_int32), ("n_inliers", ctypes.c_int64),
                ("n_keep", ctypes.c_int64), ("plane", ctypes.c_float * 4), ("refined", ctypes.c_double * 4)]


class ApResult(ctypes.Structure):
    """fec_ap_result_t (include/fec_metrics.h)."""
    _fields_ = [("tp", ctypes.c_int64), ("fp", ctypes.c_int64), ("n_pred", ctypes.c_int64),
                ("n_gt", ctypes.c_int64), ("ap", ctypes.c_double), ("status", ctypes.c_int32),
                ("pad", ctypes.c_int32)]


class FecError(RuntimeError):
    def __init__(self, code: int, detail: str):
        super().__init__(f"{_status_string(code)}: {detail}")
        self.code = code


_lib = None


def lib():
    """Load libfec.so (raises if it has not been built: no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing; run __graft_entry__.build() "
                              "(the FEC path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        i64, f32, vp, sz = ctypes.c_int64, ctypes.c_float, ctypes.c_void_p, ctypes.c_size_t
        L.fec_workspace_bytes.restype = sz
        L.fec_workspace_bytes.argtypes = [i64]
        L.fec_workspace_bytes_host.restype = sz
        L.fec_workspace_bytes_host.argtypes = [i64]
        L.fec_cluster_ws.restype = ctypes.c_int32
        L.fec_cluster_ws.argtypes = [vp, i64, f32, i64, i64, vp, vp, sz, vp]
        L.fec_cluster.restype = ctypes.c_int32
        L.fec_cluster.argtypes = [vp, i64, f32, i64, i64, vp]
        L.fec_cluster_async.restype = ctypes.c_int32
        L.fec_cluster_async.argtypes = [vp, i64, f32, i64, i64, vp, vp, vp]
        L.fec_cluster_ws_async.restype = ctypes.c_int32
        L.fec_cluster_ws_async.argtypes = [vp, i64, f32, i64, i64, vp, vp, sz, vp, vp]
        L.fec_max_points.restype = i64
        L.fec_max_points.argtypes = []
        L.fec_debug_alloc_extra.restype = None
        L.fec_debug_alloc_extra.argtypes = [sz]
        L.fec_cluster_host.restype = ctypes.c_int32
        L.fec_cluster_host.argtypes = [vp, i64, f32, i64, i64, vp, vp, sz, vp]
        L.fec_cluster_host_async.restype = ctypes.c_int32
        L.fec_cluster_host_async.argtypes = [vp, i64, f32, i64, i64, vp, vp, sz, vp, vp]
        L.fec_get_stats.restype = ctypes.c_int32
        L.fec_get_stats.argtypes = [ctypes.POINTER(FecStats)]
        L.fec_set_instrumentation.restype = None
        L.fec_set_instrumentation.argtypes = [ctypes.c_int]
        L.fec_status_string.restype = ctypes.c_char_p
        L.fec_status_string.argtypes = [ctypes.c_int32]
        L.fec_last_error.restype = ctypes.c_char_p
        L.fec_last_error.argtypes = []
        L.fec_version.restype = ctypes.c_char_p
        L.fec_version.argtypes = []
        L.fec_batch_workspace_bytes.restype = sz
        L.fec_batch_workspace_bytes.argtypes = [i64, ctypes.c_int32]
        L.fec_cluster_batch_ws.restype = ctypes.c_int32
        L.fec_cluster_batch_ws.argtypes = [vp, vp, ctypes.c_int32, f32, i64, i64, vp, vp, sz, vp]
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.fec_debug_subcell_tables.restype = ctypes.c_int32
        L.fec_debug_subcell_tables.argtypes = [u64p, u64p]
        L.fec_debug_subcell_dilate.restype = ctypes.c_uint64
        L.fec_debug_subcell_dilate.argtypes = [ctypes.c_uint64]
        L.fec_debug_subcell_components.restype = ctypes.c_int32
        L.fec_debug_subcell_components.argtypes = [ctypes.c_uint64, u64p]
        L.fec_set_item_cap.restype = None
        L.fec_set_item_cap.argtypes = [i64]
        L.fec_set_grid_mode.restype = None
        L.fec_set_grid_mode.argtypes = [ctypes.c_int]
        L.fec_set_timing.restype = None
        L.fec_set_timing.argtypes = [ctypes.c_int]
        L.fec_get_stage_times.restype = ctypes.c_int32
        L.fec_get_stage_times.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.c_int32]
        L.fec_stage_name.restype = ctypes.c_char_p
        L.fec_stage_name.argtypes = [ctypes.c_int32]
        L.fec_slab_record_words.restype = i64
        L.fec_slab_record_words.argtypes = [i64]
        L.fec_slab_workspace_bytes.restype = sz
        L.fec_slab_workspace_bytes.argtypes = [i64, ctypes.c_int32, i64]
        L.fec_slab_local.restype = ctypes.c_int32
        L.fec_slab_local.argtypes = [vp, vp, i64, i64, i64, f32, vp, i64, vp, sz, ctypes.POINTER(SlabState), vp, vp]
        L.fec_part_workspace_bytes.restype = sz
        L.fec_part_workspace_bytes.argtypes = []
        L.fec_part_max_layers.restype = ctypes.c_int32
        L.fec_part_max_layers.argtypes = []
        L.fec_part_bbox.restype = ctypes.c_int32
        L.fec_part_bbox.argtypes = [vp, i64, vp, vp, vp, sz, vp]
        L.fec_part_hist.restype = ctypes.c_int32
        L.fec_part_hist.argtypes = [vp, i64, vp, f32, vp, vp, sz, vp]
        L.fec_part_plan.restype = ctypes.c_int32
        L.fec_part_plan.argtypes = [vp, ctypes.c_int32, vp, vp, sz, vp]
        L.fec_part_pack.restype = ctypes.c_int32
        L.fec_part_pack.argtypes = [vp, vp, i64, vp, f32, vp, ctypes.c_int32, vp, vp, vp, vp, sz, vp]
        L.fec_part_order.restype = ctypes.c_int32
        L.fec_part_order.argtypes = [vp, vp, i64, vp, f32, vp, ctypes.c_int32, ctypes.c_int32, vp, vp, vp, vp, sz, vp]
        L.fec_slab_merge.restype = ctypes.c_int32
        L.fec_slab_merge.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, i64, i64, vp, vp, sz,
                                     ctypes.POINTER(SlabState), vp]
        L.fec_ground_workspace_bytes.restype = sz
        L.fec_ground_workspace_bytes.argtypes = [i64, ctypes.c_int32]
        L.fec_ground_remove.restype = ctypes.c_int32
        L.fec_ground_remove.argtypes = [vp, i64, vp, ctypes.c_int32, f32, ctypes.c_double, i64, vp, vp, vp, vp,
                                        vp, sz, vp]
        L.fec_ap_workspace_bytes.restype = sz
        L.fec_ap_workspace_bytes.argtypes = [i64]
        L.fec_average_precision.restype = ctypes.c_int32
        L.fec_average_precision.argtypes = [vp, vp, i64, ctypes.c_double, vp, vp, sz, vp]
        L.fec_ground_count_ms.restype = ctypes.c_int32
        L.fec_ground_count_ms.argtypes = [ctypes.POINTER(ctypes.c_float)]
        L.fec_ground_expand_labels.restype = ctypes.c_int32
        L.fec_ground_expand_labels.argtypes = [vp, vp, vp, i64, vp, vp]
        L.fec_debug_pred.restype = ctypes.c_int32
        L.fec_debug_pred.argtypes = [vp, vp, i64, f32, vp, vp, vp]
        _lib = L
    return _lib


def _status_string(code: int) -> str:
    try:
        return lib().fec_status_string(code).decode()
    except Exception:  # pragma: no cover
        return str(code)


def _check(code: int):
    if code != OK:
        raise FecError(code, lib().fec_last_error().decode())


def _torch():
    import torch
    return torch


def workspace_bytes(n: int) -> int:
    return int(lib().fec_workspace_bytes(int(n)))


def workspace_bytes_host(n: int) -> int:
    return int(lib().fec_workspace_bytes_host(int(n)))


def _f32(d_th: float) -> float:
    # the C ABI takes d_th as fp32; round here so callers and the oracle see the same value
    return float(np.float32(d_th))


def _stream_for(dev, stream):
    """(stream, foreign): the stream to enqueue on and whether it differs from the current one."""
    torch = _torch()
    cur = torch.cuda.current_stream(dev)
    st = stream if stream is not None else cur
    return st, st.cuda_stream != cur.cuda_stream


def _enter(st, foreign):
    """Before enqueueing on a foreign stream: order it after the current stream's pending work
    (the input tensors, and the allocations made below, were produced there)."""
    if foreign:
        st.wait_stream(_torch().cuda.current_stream(st.device))


def _keep(st, foreign, *tensors):
    """After enqueueing on a foreign stream: tensors allocated on the current stream must not be
    recycled by the caching allocator while `st` still uses them."""
    if foreign:
        for t in tensors:
            if t is not None and hasattr(t, "record_stream") and t.is_cuda:
                t.record_stream(st)


def raise_status(status) -> None:
    """Raise FecError if a device status word (int32 CUDA tensor, filled by an async call) holds
    an error.  One device->host read (synchronises with the stream that wrote it)."""
    code = int(status.item())
    if code != OK:
        raise FecError(code, {ERR_NONFINITE: "non-finite coordinate (reading A12)",
                              ERR_GRID_RANGE: "bbox extent / cell >= 2^20 on an axis (reading A14)"}.get(
                                  code, "device-side error"))


def cluster(points, d_th: float, min_size: int = 1, max_size: int = 2**62, out=None,
            workspace=None, stream=None, status=None, check: bool = True):
    """Labels of `points` (CUDA float32 tensor [n, 3], contiguous) on the current device.

    Returns an int32 CUDA tensor [n]: min input index of the point's component, or -1
    when the component size is outside [min_size, max_size].  Enqueued on PyTorch's
    current stream (or `stream`) through fec_cluster_ws_async: no host round trip, so the
    call can be captured in a CUDA graph.  `status` (int32 CUDA tensor [1], optional)
    receives the device status; with check=True (default) it is read back after the call
    (one synchronisation) and an error raises FecError."""
    torch = _torch()
    if not (isinstance(points, torch.Tensor) and points.is_cuda):
        raise TypeError("points must be a CUDA tensor (use cluster_host for host arrays)")
    if points.dtype != torch.float32 or points.dim() != 2 or points.shape[1] != 3:
        raise TypeError("points must be float32 [n, 3]")
    st, foreign = _stream_for(points.device, stream)
    points_c = points.contiguous()
    n = points_c.shape[0]
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=points.device)
    if n == 0:
        _check(lib().fec_cluster_ws(None, 0, _f32(d_th), int(min_size), int(max_size), None, None, 0, None))
        return out
    nb = workspace_bytes(n)
    if workspace is None or workspace.numel() < nb:
        workspace = torch.empty(nb, dtype=torch.uint8, device=points.device)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=points.device)
    _enter(st, foreign)
    _check(lib().fec_cluster_ws_async(points_c.data_ptr(), n, _f32(d_th), int(min_size), int(max_size),
                                      out.data_ptr(), workspace.data_ptr(), workspace.numel(), st.cuda_stream,
                                      status.data_ptr()))
    _keep(st, foreign, points_c, out, workspace, status)
    if check:
        st.synchronize()
        raise_status(status)
    return out


def cluster_async(points, d_th: float, min_size: int, max_size: int, out, status, stream=None):
    """fec_cluster_async (SURVEY §8(b)'s signature): the library takes its workspace from the
    device's stream-ordered memory pool; nothing is synchronised; `status` (int32 CUDA [1])
    receives the device status.  Graph-capturable."""
    torch = _torch()
    st, foreign = _stream_for(points.device, stream)
    n = points.shape[0]
    _enter(st, foreign)
    _check(lib().fec_cluster_async(points.data_ptr() if n else None, n, _f32(d_th), int(min_size), int(max_size),
                                   out.data_ptr() if n else None, st.cuda_stream, status.data_ptr()))
    _keep(st, foreign, points, out, status)
    return out


def cluster_host(points, d_th: float, min_size: int = 1, max_size: int = 2**62, out=None,
                 workspace=None, stream=None, device=None, sync: bool = True, status=None):
    """End-to-end form: host float32 [n, 3] in (numpy or CPU tensor; pinned memory gives
    asynchronous copies), host int32 [n] labels out.  The host<->device copies run inside
    the C ABI call (fec_cluster_host).  sync=False (fec_cluster_host_async) returns once the
    work is enqueued on `stream`: `out` is valid after the stream completes, and the caller
    keeps `points`, `out` and `workspace` alive until then (pipelining over two streams);
    `status` (int32 CUDA [1], optional) then receives the device status."""
    torch = _torch()
    if isinstance(points, torch.Tensor):
        if points.is_cuda:
            raise TypeError("cluster_host takes host memory")
        p = points.contiguous()
        n = p.shape[0]
        ptr = p.data_ptr()
        keep = p
    else:
        p = np.ascontiguousarray(points, dtype=np.float32).reshape(-1, 3)
        n = p.shape[0]
        ptr = p.ctypes.data
        keep = p
    if out is None:
        out = np.empty(n, dtype=np.int32)
    out_ptr = out.data_ptr() if isinstance(out, torch.Tensor) else out.ctypes.data
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    nb = workspace_bytes_host(n)
    if n and (workspace is None or workspace.numel() < nb):
        workspace = torch.empty(nb, dtype=torch.uint8, device=dev)
    st, foreign = _stream_for(dev, stream)
    _enter(st, foreign)
    args = (ptr if n else None, n, _f32(d_th), int(min_size), int(max_size), out_ptr if n else None,
            workspace.data_ptr() if n else None, workspace.numel() if n else 0, st.cuda_stream)
    if sync:
        _check(lib().fec_cluster_host(*args))
    else:
        if status is None and n:
            status = torch.empty(1, dtype=torch.int32, device=dev)
        _check(lib().fec_cluster_host_async(*args, status.data_ptr() if n else None))
        _keep(st, foreign, workspace, status)
    del keep
    return out


def batch_workspace_bytes(n_total: int, nclouds: int) -> int:
    return int(lib().fec_batch_workspace_bytes(int(n_total), int(nclouds)))


def cluster_batch(points, offsets, d_th: float, min_size: int = 1, max_size: int = 2**62, out=None,
                  workspace=None, stream=None):
    """Many independent clouds in one call (the paper's per-scan mode).  `points`: CUDA float32
    [n_total, 3], cloud c = rows offsets[c]:offsets[c+1] (`offsets`: host ints, nclouds + 1).
    Returns int32 CUDA labels [n_total]: minimum index inside the point's own cloud of its
    component, or -1 (size outside [min_size, max_size] within that cloud)."""
    torch = _torch()
    if not (isinstance(points, torch.Tensor) and points.is_cuda and points.dtype == torch.float32):
        raise TypeError("points must be a CUDA float32 tensor [n, 3]")
    points = points.contiguous()
    off = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
    nc = len(off) - 1
    n = points.shape[0]
    if nc < 1 or off[-1] != n:
        raise ValueError("offsets must have nclouds + 1 entries ending at len(points)")
    if out is None:
        out = torch.empty(n, dtype=torch.int32, device=points.device)
    nb = max(batch_workspace_bytes(n, nc), 1)
    if workspace is None or workspace.numel() < nb:
        workspace = torch.empty(nb, dtype=torch.uint8, device=points.device)
    st, foreign = _stream_for(points.device, stream)
    _enter(st, foreign)
    _check(lib().fec_cluster_batch_ws(_ptr(points), off.ctypes.data, nc, _f32(d_th), int(min_size), int(max_size),
                                      _ptr(out), workspace.data_ptr(), workspace.numel(), st.cuda_stream))
    _keep(st, foreign, points, out, workspace)
    return out


# ---- ground removal (include/fec_ground.h) ----------------------------
GROUND_RESULT_BYTES = ctypes.sizeof(GroundResult)


def ground_workspace_bytes(n: int, n_hyp: int) -> int:
    return int(lib().fec_ground_workspace_bytes(int(n), int(n_hyp)))


def ground_result(buf) -> dict:
    """Decode a device fec_ground_result_t (uint8 CUDA tensor) -- a device->host read."""
    raw = bytes(buf[:GROUND_RESULT_BYTES].cpu().numpy().tobytes())
    r = GroundResult.from_buffer_copy(raw)
    return {"best": r.best, "n_valid": r.n_valid, "n_inliers": r.n_inliers, "n_keep": r.n_keep,
            "plane": np.array(list(r.plane), dtype=np.float32), "refined": np.array(list(r.refined))}


def remove_ground(points, triplets, threshold: float = 0.2, max_tilt_deg: float = 30.0, min_inliers=None,
                  cos_max_tilt=None, out=None, workspace=None, stream=None, counts=False):
    """RANSAC plane-fit ground removal on the device.  `points`: CUDA float32 [n, 3];
    `triplets`: CUDA int32 [H, 3] point indices per hypothesis (the caller's random sample).
    Returns (keep_points [n, 3], keep_idx [n], result_buf, counts_or_None): the first
    n_keep rows are the survivors in input order; `result_buf` holds fec_ground_result_t on
    the device (ground_result() reads it).  Nothing is synchronised."""
    import math
    torch = _torch()
    if not (isinstance(points, torch.Tensor) and points.is_cuda and points.dtype == torch.float32):
        raise TypeError("points must be a CUDA float32 tensor [n, 3]")
    if not (isinstance(triplets, torch.Tensor) and triplets.is_cuda and triplets.dtype == torch.int32):
        raise TypeError("triplets must be a CUDA int32 tensor [H, 3]")
    points = points.contiguous()
    triplets = triplets.contiguous()
    n, H = points.shape[0], triplets.numel() // 3
    if min_inliers is None:
        min_inliers = (n + 9) // 10
    if cos_max_tilt is None:
        cos_max_tilt = math.cos(math.radians(max_tilt_deg))
    dev = points.device
    if out is None:
        out = (torch.empty((max(n, 1), 3), dtype=torch.float32, device=dev),
               torch.empty(max(n, 1), dtype=torch.int32, device=dev),
               torch.empty(GROUND_RESULT_BYTES, dtype=torch.uint8, device=dev))
    kp, ki, res = out
    cnt = torch.empty(max(H, 1), dtype=torch.int64, device=dev) if counts else None
    nb = ground_workspace_bytes(n, H)
    if nb == 0:
        raise FecError(ERR_INVALID_ARGUMENT, "bad sizes for fec_ground_remove")
    if workspace is None or workspace.numel() < nb:
        workspace = torch.empty(nb, dtype=torch.uint8, device=dev)
    st, foreign = _stream_for(dev, stream)
    _enter(st, foreign)
    _check(lib().fec_ground_remove(_ptr(points) if n else None, n, _ptr(triplets) if H else None, H,
                                   float(np.float32(threshold)), float(cos_max_tilt), int(min_inliers),
                                   _ptr(kp), _ptr(ki), _ptr(cnt) if cnt is not None else None, _ptr(res),
                                   workspace.data_ptr(), workspace.numel(), st.cuda_stream))
    _keep(st, foreign, points, triplets, kp, ki, res, cnt, workspace)
    return kp, ki, res, cnt


def ground_count_ms() -> float:
    """Duration of the last fec_ground_remove's inlier-counting kernel (needs set_timing(True))."""
    v = ctypes.c_float(-1.0)
    _check(lib().fec_ground_count_ms(ctypes.byref(v)))
    return float(v.value)


def expand_labels(keep_idx, keep_labels, result_buf, n: int, out=None, stream=None):
    """Whole-cloud labels from the survivors' labels: -2 = ground, -1 = noise, else the
    input-order minimum index of the point's cluster (fec_ground_expand_labels)."""
    torch = _torch()
    dev = keep_idx.device
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    st, foreign = _stream_for(dev, stream)
    _enter(st, foreign)
    _check(lib().fec_ground_expand_labels(_ptr(keep_idx), _ptr(keep_labels), _ptr(result_buf), int(n), _ptr(out),
                                          st.cuda_stream))
    _keep(st, foreign, keep_idx, keep_labels, result_buf, out)
    return out[:n]


def cluster_nonground(points, triplets, d_th: float, min_size: int = 1, max_size: int = 2**62,
                      threshold: float = 0.2, max_tilt_deg: float = 30.0, min_inliers=None):
    """Ground removal then clustering of the survivors ("(i) ground points
    removal and (ii) the clustering of the remaining points").  One device->host read of
    n_keep between the two.  Returns (labels [n] int32 CUDA: -2 ground / -1 noise / cluster
    min index, result dict)."""
    kp, ki, res, _ = remove_ground(points, triplets, threshold, max_tilt_deg, min_inliers)
    info = ground_result(res)
    nk = int(info["n_keep"])
    lab_k = cluster(kp[:nk], d_th, min_size, max_size)
    return expand_labels(ki, lab_k, res, points.shape[0]), info


# ---- AP metric (include/fec_metrics.h) ---------------------------------
AP_RESULT_BYTES = ctypes.sizeof(ApResult)


def ap_workspace_bytes(n: int) -> int:
    return int(lib().fec_ap_workspace_bytes(int(n)))


def average_precision(pred, gt, threshold: float = 0.75, workspace=None, stream=None, result=None,
                      read: bool = True):
    """AP of predicted labels `pred` (CUDA int32 [n]: -1 or a point index) against ground truth
    `gt` (CUDA int32 [n] in [0, n], 0 = unlabelled).  Returns a dict (one device->host read)
    or, with read=False, the device result buffer."""
    torch = _torch()
    for t in (pred, gt):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.int32):
            raise TypeError("pred and gt must be CUDA int32 tensors")
    if pred.numel() != gt.numel():
        raise ValueError("pred and gt must cover the same cloud")
    pred, gt = pred.contiguous(), gt.contiguous()
    n = pred.numel()
    dev = pred.device
    nb = ap_workspace_bytes(n)
    if workspace is None or workspace.numel() < nb:
        workspace = torch.empty(nb, dtype=torch.uint8, device=dev)
    if result is None:
        result = torch.empty(AP_RESULT_BYTES, dtype=torch.uint8, device=dev)
    st, foreign = _stream_for(dev, stream)
    _enter(st, foreign)
    _check(lib().fec_average_precision(_ptr(pred), _ptr(gt), n, float(threshold), result.data_ptr(),
                                       workspace.data_ptr(), workspace.numel(), st.cuda_stream))
    _keep(st, foreign, pred, gt, workspace, result)
    if not read:
        return result
    if foreign:  # the read below runs on the current stream: order it after the kernels on `st`
        torch.cuda.current_stream(dev).wait_stream(st)
    r = ApResult.from_buffer_copy(bytes(result.cpu().numpy().tobytes()))
    return {"tp": r.tp, "fp": r.fp, "n_pred": r.n_pred, "n_gt": r.n_gt, "ap": r.ap, "status": r.status}


def set_instrumentation(enable: bool):
    lib().fec_set_instrumentation(1 if enable else 0)


def stats() -> dict:
    s = FecStats()
    _check(lib().fec_get_stats(ctypes.byref(s)))
    d = {k: getattr(s, k) for k, _ in FecStats._fields_ if k != "dims"}
    d["dims"] = list(s.dims)
    return d


def set_grid_mode(mode: int):
    """Testing aid: 0 = automatic, 1 = hashed cell index (open-addressing table of occupied
    cells) always, 2 = key sort (bitmap index), 3 = counting sort (bitmap index)."""
    lib().fec_set_grid_mode(int(mode))


def debug_alloc_extra(nbytes: int):
    """Testing aid: self-allocating calls ask for `nbytes` more (a huge value forces
    FEC_ERR_OUT_OF_MEMORY); 0 turns it off."""
    lib().fec_debug_alloc_extra(int(nbytes))


def set_item_cap(cap: int):
    """Testing aid: cap the queued uncertain dense pairs (0 = default); labels do not change."""
    lib().fec_set_item_cap(int(cap))


def set_timing(enable: bool):
    lib().fec_set_timing(1 if enable else 0)


def stage_times() -> dict:
    """{stage name: ms} of this thread's last timed call (waits for its last event)."""
    buf = (ctypes.c_float * 16)()
    k = lib().fec_get_stage_times(buf, 16)
    if k < 0:
        raise FecError(ERR_INVALID_ARGUMENT, lib().fec_last_error().decode())
    return {lib().fec_stage_name(i).decode(): float(buf[i]) for i in range(k)}


def debug_pred(a, b, d_th: float):
    """Device predicate on pairs (CUDA float32 [m,3] tensors) -> (bool tensor, d2 tensor)."""
    torch = _torch()
    m = a.shape[0]
    out = torch.empty(m, dtype=torch.uint8, device=a.device)
    d2 = torch.empty(m, dtype=torch.float32, device=a.device)
    st = torch.cuda.current_stream(a.device)
    _check(lib().fec_debug_pred(a.contiguous().data_ptr(), b.contiguous().data_ptr(), m, _f32(d_th),
                                out.data_ptr(), d2.data_ptr(), st.cuda_stream))
    return out.bool(), d2


# ---- multi-GPU slab path (include/fec.h "Multi-GPU slab path"; driver in .dist) ---------------
def slab_record_words(rec_cap: int) -> int:
    return int(lib().fec_slab_record_words(int(rec_cap)))


def slab_workspace_bytes(n_local: int, world: int, rec_cap: int) -> int:
    return int(lib().fec_slab_workspace_bytes(int(n_local), int(world), int(rec_cap)))


def _ptr(t):
    return t.data_ptr() if t is not None and t.numel() else None


def slab_local(points, gidx, n_owned: int, n_first: int, d_th: float, records, rec_cap: int, workspace,
               stream=None, status=None) -> SlabState:
    """Step 1 on this rank: cluster owned ∪ halo (CUDA float32 [n_local, 3], local order
    first-layer | other owned | halo) and pack boundary records into `records` (CUDA int32
    [slab_record_words(rec_cap)]).  Returns the state slab_merge needs."""
    torch = _torch()
    if not (isinstance(points, torch.Tensor) and points.is_cuda and points.dtype == torch.float32):
        raise TypeError("points must be a CUDA float32 tensor [n, 3]")
    if gidx.dtype != torch.int32 or records.dtype != torch.int32 or not gidx.is_cuda or not records.is_cuda:
        raise TypeError("gidx and records must be CUDA int32 tensors")
    points = points.contiguous()
    n_local = points.shape[0]
    st, foreign = _stream_for(records.device, stream)
    _enter(st, foreign)
    state = SlabState()
    _check(lib().fec_slab_local(_ptr(points), _ptr(gidx), n_local, int(n_owned), int(n_first), _f32(d_th),
                                records.data_ptr(), int(rec_cap), workspace.data_ptr(), workspace.numel(),
                                ctypes.byref(state), st.cuda_stream, _ptr(status)))
    _keep(st, foreign, points, gidx, records, workspace, status)
    return state


def slab_merge(all_records, world: int, rank: int, min_size: int, max_size: int, labels_owned, workspace,
               state: SlabState, stream=None):
    """Step 3 on this rank: replicated boundary union-find over the gathered records, then
    the global labels (min global index, or -1) of the rank's owned points."""
    torch = _torch()
    st, foreign = _stream_for(all_records.device, stream)
    _enter(st, foreign)
    _check(lib().fec_slab_merge(all_records.data_ptr(), int(world), int(rank), int(min_size), int(max_size),
                                _ptr(labels_owned), workspace.data_ptr(), workspace.numel(), ctypes.byref(state),
                                st.cuda_stream))
    return labels_owned


def subcell_tables():
    """(certain, reach) uint64 arrays [27, 64] of the dense path's sub-cell relations (host)."""
    c = np.zeros(27 * 64, np.uint64)
    r = np.zeros(27 * 64, np.uint64)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib().fec_debug_subcell_tables(c.ctypes.data_as(u64p), r.ctypes.data_as(u64p))
    return c.reshape(27, 64), r.reshape(27, 64)


def subcell_dilate(m: int) -> int:
    return int(lib().fec_debug_subcell_dilate(int(m)))


def subcell_components(occ: int):
    out = np.zeros(8, np.uint64)
    k = lib().fec_debug_subcell_components(int(occ), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return [int(x) for x in out[:k]] if k >= 0 else None
