"""Build libfsw.so in-tree: all CUDA kernels for sm_100a + the C++ host runtime.

    python -m paper_2306_03622_b200.build          # incremental
    python -m paper_2306_03622_b200.build --force

nvcc cross-compiles for sm_100a without a GPU.  The .so is git-ignored but travels to the
GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
SO = os.path.join(PKG, "libfsw.so")
SO_TRACE = os.path.join(PKG, "libfsw_trace.so")
BUILD = os.path.join(PKG, "_build")

CU_SOURCES = ["swap.cu", "ops.cu", "gemm_tc.cu", "gemm_ws.cu", "attn_tc.cu", "mega.cu"]
CXX_SOURCES = ["runtime.cpp", "store.cpp", "plan.cpp", "graph.cpp", "invoke.cpp", "sched.cpp", "litmus.cpp"]
HEADERS = ["kernels.h", "device.cuh", "policy.h", "rt_internal.h", "umma.cuh", "attn_core.cuh"]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-Wno-deprecated-gpu-targets", "-O3", "-std=c++17", "-lineinfo", f"-I{INCLUDE}", f"-I{CSRC}", "-Xcompiler", "-fPIC"]


def _stale(obj, deps):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> str:
    """libfsw.so; trace=True builds libfsw_trace.so, the same library with the device-timeline stamps compiled
    into the kernels (FSW_TRACE_KERNELS; load it with FSW_LIB=libfsw_trace.so, tools/timeline.py)."""
    build_dir = BUILD + ("_trace" if trace else "")
    so = SO_TRACE if trace else SO
    extra = ["-DFSW_TRACE_KERNELS"] if trace else []
    os.makedirs(build_dir, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "fsw.h")]
    objs = []
    for src in CU_SOURCES + CXX_SOURCES:
        path = os.path.join(CSRC, src)
        obj = os.path.join(build_dir, src + ".o")
        objs.append(obj)
        if force or _stale(obj, [path] + hdrs):
            cmd = [NVCC] + ARCH + COMMON + extra + ["-c", path, "-o", obj]
            if src.endswith(".cu"):
                cmd += ["-Xptxas", "-v"] if verbose else []
            else:
                cmd = [NVCC] + COMMON + extra + ["-x", "c++", "-c", path, "-o", obj]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or _stale(so, objs):
        cmd = [NVCC] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", so] + objs
        subprocess.check_call(cmd)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv, trace="--trace" in sys.argv))
