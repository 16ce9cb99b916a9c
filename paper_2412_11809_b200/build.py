"""Build libtpxcluster.so (the C-ABI library) for sm_100a with nvcc.

The library is plain CUDA C++ behind ``include/tpx_cluster.h``; it links the
CUDA runtime statically and NCCL dynamically (sharded path).  Built in-tree
so the .so travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libtpxcluster.so")
# bounds-checked build (device asserts, -DTPX_CHECKED): tests only
CHECKED_LIB = os.path.join(LIBDIR, "checked", "libtpxcluster.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "--expt-relaxed-constexpr",
              "-Xptxas", "-v"]


def _nvcc() -> str:
    for cand in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.isabs(cand) and os.path.exists(cand):
            return cand
    return "nvcc"


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + glob.glob(os.path.join(INCLUDE, "*.h")))


def needs_build(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(s) > t for s in _sources())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """Compile the library if any source is newer than the .so.  checked=True
    builds the bounds-checked variant (TPX_BOUND device asserts) into
    lib/checked/ instead; the product never loads it."""
    lib = CHECKED_LIB if checked else LIB
    if not force and not needs_build(lib):
        return lib
    os.makedirs(os.path.dirname(lib), exist_ok=True)
    tus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    tmp = lib + f".tmp{os.getpid()}"
    extra = ["-DTPX_CHECKED"] if checked else []
    cmd = [_nvcc(), *ARCH, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-shared", "-o", tmp, *tus]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {lib}")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
