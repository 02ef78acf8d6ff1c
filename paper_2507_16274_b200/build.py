"""Build libstw.so (sm_100a) in-tree with nvcc; no JIT, no torch extension cache."""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libstw.so")
ALLOC_LIB = os.path.join(PKG, "libstw_alloc.so")
ALLOC_SRC = os.path.join(PKG, "csrc_alloc", "stw_alloc.cpp")
IO_LIB = os.path.join(PKG, "libstw_io.so")
IO_SRC = os.path.join(PKG, "csrc_io", "stw_io.cpp")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = [
    "-O3", "-lineinfo", "-std=c++17", "--fmad=false", "-Xcompiler", "-fPIC,-ffp-contract=off",
    "-shared", "-cudart", "static", "-I" + os.path.join(ROOT, "include"),
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "stw.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"build failed: {cmd[-1]}")


def build_alloc(force: bool = False, verbose: bool = False) -> str:
    """libstw_alloc.so: the CUDAPluggableAllocator (host C++ + cudart)."""
    deps = [ALLOC_SRC, os.path.join(ROOT, "include", "stw_alloc.h"), os.path.join(ROOT, "include", "stw.h")]
    if force or not os.path.exists(ALLOC_LIB) or any(os.path.getmtime(p) > os.path.getmtime(ALLOC_LIB) for p in deps):
        _run([NVCC, "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
              "-I" + os.path.join(ROOT, "include"), "-o", ALLOC_LIB, ALLOC_SRC], verbose)
    return ALLOC_LIB


def build_io(force: bool = False, verbose: bool = False) -> str:
    """libstw_io.so: trace / plan files (host C++ only)."""
    deps = [IO_SRC, os.path.join(ROOT, "include", "stw_io.h"), os.path.join(ROOT, "include", "stw.h")]
    if force or not os.path.exists(IO_LIB) or any(os.path.getmtime(p) > os.path.getmtime(IO_LIB) for p in deps):
        _run(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-Wall", "-I" + os.path.join(ROOT, "include"), "-o",
              IO_LIB, IO_SRC], verbose)
    return IO_LIB


def build(force: bool = False, verbose: bool = False) -> str:
    build_alloc(force, verbose)
    build_io(force, verbose)
    if force or stale():
        extra = os.environ.get("STW_NVCC_EXTRA", "").split()  # e.g. -DSTW_REPLAY_CLOCK (diagnostic builds)
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-o", LIB, *sources()]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("nvcc failed building libstw.so")
        if verbose and (res.stdout or res.stderr):
            sys.stderr.write(res.stdout + res.stderr)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
