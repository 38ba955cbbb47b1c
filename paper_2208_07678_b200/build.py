"""Build libfec.so (the C-ABI library) in-tree for sm_100a with nvcc.

No fast-math, no FMA contraction (-fmad=false), no flush-to-zero: the fp32 predicate of
Eq. 1 must round every operation (readings A2/A3)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(HERE, "libfec.so")
SOURCES = ["fec_capi.cu", "fec_kernels.cu", "fec_dense.cu", "fec_sort.cu", "fec_scan_prim.cu", "fec_slab.cu", "fec_part.cu", "fec_ground.cu", "fec_metrics.cu"]
HEADERS = ["fec_internal.cuh", "fec_kernels.cuh", "fec_slab.cuh", "fec_subcell.cuh", "fec_part.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false", "-ftz=false", "-prec-div=true", "-prec-sqrt=true",
    "-Xcompiler", "-fPIC,-ffp-contract=off,-fno-fast-math",
    "-Xptxas", "-v",
] + [f"-D{k}={v}" for k, v in (("FEC_UF_RELAXED", os.environ.get("FEC_UF_RELAXED")),) if v is not None]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(INCLUDE, "fec.h"), os.path.join(INCLUDE, "fec_ground.h"), os.path.join(INCLUDE, "fec_metrics.h"), __file__]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    os.makedirs(os.path.join(HERE, "_obj"), exist_ok=True)
    for s in SOURCES:
        o = os.path.join(HERE, "_obj", s.replace(".cu", ".o"))
        cmd = [NVCC, *NVCC_FLAGS, "-I", INCLUDE, "-I", CSRC, "-c", os.path.join(CSRC, s), "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {s}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(o)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
