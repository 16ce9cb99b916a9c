"""Parallel multi-core CPU comparator.

The paper's CPU method -- temporal splitting into time windows processed by
worker threads round-robin, Alg. 1 per window with the per-pixel reference
matrix, and the merge cascade for border clusters (§3.2.3
l.117-119, §3.3 l.121-139) -- in plain C with pthreads
(``tpx_cpu_parallel.c``).  A baseline timed beside the GPU path and the
single-threaded oracle in ``bench.py``; it shares no code with either.  Its
output contract is tpx_cluster_run's (labels = smallest input index,
64-byte records in ascending label order), checked against the oracle in
``tests/test_cpu_parallel.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tpx_cpu_parallel.c")
_LIB = os.path.join(_HERE, "libtpxcpupar.so")

FEAT_DTYPE = np.dtype(
    [("label", "<u4"), ("size", "<u4"), ("toa_min", "<u8"), ("toa_max", "<u8"),
     ("tot_sum", "<u8"), ("sum_x", "<u8"), ("sum_y", "<u8"), ("sum_tot_x", "<u8"),
     ("sum_tot_y", "<u8")]
)


class _Stats(ctypes.Structure):
    _fields_ = [(k, ctypes.c_uint64) for k in ("windows", "clusters", "border_clusters", "border_checks",
                                               "bbox_checks", "full_checks", "merges")]


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-shared", "-fPIC", "-std=gnu11", "-pthread", "-o", tmp,
                               _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        L.cpu_parallel_cluster.argtypes = [vp, u64, u64, u32, u32, u64, ctypes.c_int, vp, vp, ctypes.POINTER(u64),
                                           ctypes.POINTER(_Stats)]
        L.cpu_parallel_cluster.restype = ctypes.c_int
        _lib = L
    return _lib


def cluster(hits, dt: int, width: int = 256, height: int = 256, threads: int | None = None,
            window_ticks: int = 0, stats: bool = False):
    """Returns ``(labels uint32[n], features FEAT_DTYPE[k])`` (and a stats dict
    if ``stats``).  ``threads`` defaults to the CPUs this process may use;
    ``window_ticks`` 0 = 100 * dt_max (the paper's window >> dt_max)."""
    h = np.ascontiguousarray(hits)
    assert h.dtype.itemsize == 16
    n = len(h)
    if threads is None:
        threads = len(os.sched_getaffinity(0))
    labels = np.zeros(max(n, 1), dtype=np.uint32)
    feats = np.zeros(max(n, 1), dtype=FEAT_DTYPE)
    k = ctypes.c_uint64(0)
    st = _Stats()
    rc = _load().cpu_parallel_cluster(h.ctypes.data if n else None, n, int(dt), width, height, int(window_ticks),
                                      int(threads), labels.ctypes.data, feats.ctypes.data, ctypes.byref(k),
                                      ctypes.byref(st))
    if rc != 0:
        raise RuntimeError(f"cpu_parallel_cluster returned {rc}")
    out = (labels[:n], feats[: k.value].copy())
    if stats:
        return out + ({f: getattr(st, f) for f, _ in _Stats._fields_},)
    return out
