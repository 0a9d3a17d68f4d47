"""In-tree build of the sm_100a CUDA library (libwgpf.so).

nvcc cross-compiles for sm_100a without a GPU, so this runs in the build
container (``__graft_entry__.build()``) and the .so travels to the GPU box with
the repo snapshot.  On a box where it is missing (or stale) the loader rebuilds
it with the same command; there is no CPU fallback.
"""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "_lib")
LIB = os.path.join(LIBDIR, "libwgpf.so")
CSRC_P1 = os.path.join(PKG, "csrc_p1")
LIB_P1 = os.path.join(LIBDIR, "libwgpf_p1.so")
INCLUDE = os.path.join(ROOT, "include")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "*.cuh")) +
                  glob.glob(os.path.join(CSRC, "*.inc")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def _compile(srcs, out, log):
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = out + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, f"-I{INCLUDE}", f"-I{CSRC}", *srcs, "-o", tmp]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed building {os.path.basename(out)}:\n" +
                           res.stderr[-8000:])
    with open(os.path.join(LIBDIR, log), "w") as f:
        f.write(res.stderr)
    os.replace(tmp, out)
    return res.stderr


def p1_sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC_P1, "*.cu")) +
                  glob.glob(os.path.join(CSRC_P1, "*.cuh")) +
                  glob.glob(os.path.join(INCLUDE, "*.cuh")) +
                  glob.glob(os.path.join(INCLUDE, "*.h")))


def build(force: bool = False, verbose: bool = False) -> str:
    """libwgpf.so: the P2 post-processor (C-ABI include/wgpf.h)."""
    if force or stale():
        err = _compile([os.path.join(CSRC, "capi.cu")], LIB, "ptxas.txt")
        if verbose:
            print(err)
    return LIB


def build_p1(force: bool = False) -> str:
    """libwgpf_p1.so: P1 runtime workloads (self-test, record cost, GEMM)."""
    fresh = os.path.exists(LIB_P1) and all(
        os.path.getmtime(s) <= os.path.getmtime(LIB_P1) for s in p1_sources())
    if force or not fresh:
        _compile(sorted(glob.glob(os.path.join(CSRC_P1, "*.cu"))), LIB_P1,
                 "ptxas_p1.txt")
    return LIB_P1
