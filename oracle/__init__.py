"""FEC oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow CPU implementations of what the FEC hot path computes (see fec_oracle.c's
header for the definition and citations).  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this package.
It shares no code with the CUDA path and never imports ``paper_2208_07678_b200``.

* ``fec(points, d_th, min_size, max_size)`` — grid flood fill in C (fec_oracle.c).
* ``brute_fec(...)`` — O(n^2) definition in numpy (brute.py), for tiny inputs.
* ``Index(points, d_th).component(i)`` — (min C(i), |C(i)|) for sampled full-size parity.
* ``ground.ransac_ground(...)`` — RANSAC plane-fit ground removal (ground_oracle.c + numpy
  least-squares refinement), SURVEY §8(f) N2.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .brute import brute_fec, brute_labels_unfiltered, pred_f32, d2_f32  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fec_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "ground_oracle.c")]
_LIB = os.path.join(_HERE, "_build", "liboracle.so")

OK, ERR_INVALID_ARGUMENT, ERR_NONFINITE, ERR_RANGE, ERR_NOMEM = 0, -1, -2, -3, -4

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-shared", "-fPIC"]


def compile_oracle(force: bool = False) -> str:
    os.makedirs(os.path.dirname(_LIB), exist_ok=True)
    if force or not os.path.exists(_LIB) or any(os.path.getmtime(_LIB) < os.path.getmtime(s) for s in _SRCS):
        subprocess.check_call(["gcc", *CFLAGS, "-o", _LIB, *_SRCS, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(compile_oracle())
        f32p = ctypes.POINTER(ctypes.c_float)
        L.oracle_t2.restype = ctypes.c_float
        L.oracle_t2.argtypes = [ctypes.c_float]
        L.oracle_pred.restype = ctypes.c_int
        L.oracle_pred.argtypes = [f32p, f32p, ctypes.c_float]
        L.oracle_d2.restype = ctypes.c_float
        L.oracle_d2.argtypes = [f32p, f32p]
        L.oracle_fec.restype = ctypes.c_int
        L.oracle_fec.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_float, ctypes.c_int64,
                                 ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_index_build.restype = ctypes.c_void_p
        L.oracle_index_build.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_float,
                                         ctypes.POINTER(ctypes.c_int32)]
        L.oracle_index_free.restype = None
        L.oracle_index_free.argtypes = [ctypes.c_void_p]
        L.oracle_component.restype = ctypes.c_int
        L.oracle_component.argtypes = [ctypes.c_void_p, ctypes.c_int64,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int64)]
        i32p = ctypes.POINTER(ctypes.c_int32)
        L.oracle_ground_plane.restype = ctypes.c_int
        L.oracle_ground_plane.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_double,
                                          ctypes.c_void_p, i32p]
        L.oracle_ground_residual.restype = ctypes.c_float
        L.oracle_ground_residual.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        L.oracle_ground_counts.restype = None
        L.oracle_ground_counts.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int32,
                                           ctypes.c_float, ctypes.c_double, ctypes.c_void_p, ctypes.c_void_p,
                                           ctypes.c_void_p]
        L.oracle_ground_mask.restype = ctypes.c_int64
        L.oracle_ground_mask.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_float,
                                         ctypes.c_void_p]
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int):
        super().__init__(f"oracle error {code}")
        self.code = code


def _pts(points) -> np.ndarray:
    p = np.ascontiguousarray(points, dtype=np.float32)
    if p.ndim != 2 or (p.shape[0] and p.shape[1] != 3):
        p = p.reshape(-1, 3)
    return p


def t2(d: float) -> float:
    return float(lib().oracle_t2(ctypes.c_float(d)))


def pred(a, b, d: float) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    f32p = ctypes.POINTER(ctypes.c_float)
    return bool(lib().oracle_pred(a.ctypes.data_as(f32p), b.ctypes.data_as(f32p), t2(d)))


def d2(a, b) -> np.float32:
    a = np.ascontiguousarray(a, dtype=np.float32)
    b = np.ascontiguousarray(b, dtype=np.float32)
    f32p = ctypes.POINTER(ctypes.c_float)
    return np.float32(lib().oracle_d2(a.ctypes.data_as(f32p), b.ctypes.data_as(f32p)))


def fec(points, d_th: float, min_size: int = 1, max_size: int = 2**62, return_stats: bool = False):
    """labels[i] = min C(i) if min_size <= |C(i)| <= max_size else -1  (int32, input order)."""
    p = _pts(points)
    n = p.shape[0]
    labels = np.empty(n, dtype=np.int32)
    stats = np.zeros(2, dtype=np.int64)
    rc = lib().oracle_fec(p.ctypes.data, n, ctypes.c_float(np.float32(d_th)), int(min_size),
                          int(max_size), labels.ctypes.data, stats.ctypes.data)
    if rc != OK:
        raise OracleError(rc)
    if return_stats:
        return labels, {"components": int(stats[0]), "pred_tests": int(stats[1])}
    return labels


class Index:
    """Bucketed cloud for one-component queries: component(i) -> (min C(i), |C(i)|)."""

    def __init__(self, points, d_th: float):
        self._p = _pts(points)  # keep alive: the C side holds a pointer
        rc = ctypes.c_int32(0)
        self._h = lib().oracle_index_build(self._p.ctypes.data, self._p.shape[0],
                                           ctypes.c_float(np.float32(d_th)), ctypes.byref(rc))
        if rc.value != OK:
            raise OracleError(rc.value)

    def component(self, i: int):
        mn, sz = ctypes.c_int64(0), ctypes.c_int64(0)
        rc = lib().oracle_component(self._h, int(i), ctypes.byref(mn), ctypes.byref(sz))
        if rc != OK:
            raise OracleError(rc)
        return int(mn.value), int(sz.value)

    def close(self):
        if getattr(self, "_h", None):
            lib().oracle_index_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


def label_of(component_min: int, component_size: int, min_size: int, max_size: int) -> int:
    return component_min if min_size <= component_size <= max_size else -1
