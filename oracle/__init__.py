"""CPU oracle for Timepix3 hit clustering -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product path
(``paper_2412_11809_b200``) never imports it and shares no code with it.

All arithmetic lives in ``tpx_oracle.c`` (plain single-threaded C); this module
only compiles it with gcc and marshals numpy arrays.  See that file's header
for the definition it follows (§2 lines 29-45, §2.1 lines 61-62,
§4.1) and DESIGN.md "Readings" R1-R8.

Parity: pinned -- every function here is checked in ``tests/test_oracle_pins.py``
against brute force, hand-derived examples, scipy/networkx special cases and
invariants.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tpx_oracle.c")
_LIB = os.path.join(_HERE, "libtpxoracle.so")

#: 64-byte feature record (the layout of tpx_cluster_features).
FEAT_DTYPE = np.dtype(
    [("label", "<u4"), ("size", "<u4"), ("toa_min", "<u8"), ("toa_max", "<u8"),
     ("tot_sum", "<u8"), ("sum_x", "<u8"), ("sum_y", "<u8"), ("sum_tot_x", "<u8"),
     ("sum_tot_y", "<u8")]
)
assert FEAT_DTYPE.itemsize == 64

#: 32-byte shape record (the layout of tpx_cluster_shape).
SHAPE_DTYPE = np.dtype(
    [("x_min", "<u2"), ("x_max", "<u2"), ("y_min", "<u2"), ("y_max", "<u2"),
     ("sum_xx", "<u8"), ("sum_xy", "<u8"), ("sum_yy", "<u8")]
)
assert SHAPE_DTYPE.itemsize == 32

LOCAL, GLOBAL, STATIC = 0, 1, 2


class OracleError(RuntimeError):
    pass


def build(force: bool = False) -> str:
    """Compile libtpxoracle.so (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-std=c11", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        vp, u64, u32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32
        L.oracle_cluster_local.argtypes = [vp, u64, u64, u32, u32, vp, vp, ctypes.POINTER(u64)]
        L.oracle_cluster_local.restype = ctypes.c_int
        L.oracle_count_edges.argtypes = [vp, u64, u64, u32, u32]
        L.oracle_count_edges.restype = ctypes.c_int64
        L.oracle_index_new.argtypes = [vp, u64, u64, u32, u32]
        L.oracle_index_new.restype = vp
        L.oracle_index_delete.argtypes = [vp]
        L.oracle_index_delete.restype = None
        L.oracle_index_component.argtypes = [vp, u32, vp, u64, vp]
        L.oracle_index_component.restype = ctypes.c_int64
        L.oracle_cluster_streaming.argtypes = [vp, u64, u64, u32, u32, ctypes.c_int, vp]
        L.oracle_cluster_streaming.restype = ctypes.c_int
        L.oracle_shapes.argtypes = [vp, u64, vp, vp, u64, vp]
        L.oracle_shapes.restype = ctypes.c_int
        L.oracle_group.argtypes = [vp, u64, vp, vp, u64, vp, vp, vp]
        L.oracle_group.restype = ctypes.c_int
        L.oracle_centroids.argtypes = [vp, u64, vp]
        L.oracle_centroids.restype = None
        _lib = L
    return _lib


def _hits(h) -> np.ndarray:
    h = np.ascontiguousarray(h)
    assert h.dtype.itemsize == 16, "hits must be 16-byte tpx_hit records"
    return h


def cluster(hits, dt: int, width: int = 256, height: int = 256):
    """Connected-component clustering, variant (iii)(a).

    Returns ``(labels uint32[n], features FEAT_DTYPE[k])``; features are in
    ascending label order.
    """
    h = _hits(hits)
    n = len(h)
    labels = np.zeros(n, dtype=np.uint32)
    feats = np.zeros(max(n, 1), dtype=FEAT_DTYPE)
    k = ctypes.c_uint64(0)
    rc = _load().oracle_cluster_local(
        h.ctypes.data if n else None, n, int(dt), width, height,
        labels.ctypes.data, feats.ctypes.data, ctypes.byref(k))
    if rc != 0:
        raise OracleError(f"oracle_cluster_local returned {rc}")
    return labels, feats[: k.value].copy()


def count_edges(hits, dt: int, width: int = 256, height: int = 256) -> int:
    h = _hits(hits)
    r = _load().oracle_count_edges(h.ctypes.data if len(h) else None, len(h), int(dt), width, height)
    if r < 0:
        raise OracleError("oracle_count_edges failed")
    return int(r)


def cluster_streaming(hits, dt: int, variant: int, width: int = 256, height: int = 256) -> np.ndarray:
    """Streaming convention for variants (iii)(a/b/c); O(n^2), small n only."""
    h = _hits(hits)
    labels = np.zeros(len(h), dtype=np.uint32)
    rc = _load().oracle_cluster_streaming(
        h.ctypes.data if len(h) else None, len(h), int(dt), width, height, variant,
        labels.ctypes.data)
    if rc != 0:
        raise OracleError(f"oracle_cluster_streaming returned {rc}")
    return labels


def shapes(hits, labels, feats) -> np.ndarray:
    """Bounding box + unweighted second moments per cluster (order of feats)."""
    h = _hits(hits)
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    f = np.ascontiguousarray(feats, dtype=FEAT_DTYPE)
    out = np.zeros(max(len(f), 1), dtype=SHAPE_DTYPE)
    rc = _load().oracle_shapes(h.ctypes.data if len(h) else None, len(h), lab.ctypes.data if len(h) else None,
                               f.ctypes.data if len(f) else None, len(f), out.ctypes.data)
    if rc != 0:
        raise OracleError(f"oracle_shapes returned {rc}")
    return out[: len(f)].copy()


def group(hits, labels, feats):
    """Cluster-contiguous order (Alg. GPU Step 6, reading R18).

    Returns ``(order uint32[n], offsets uint64[k+1], cluster_of uint32[k])``.
    """
    h = _hits(hits)
    n = len(h)
    lab = np.ascontiguousarray(labels, dtype=np.uint32)
    f = np.ascontiguousarray(feats, dtype=FEAT_DTYPE)
    k = len(f)
    order = np.zeros(max(n, 1), dtype=np.uint32)
    offsets = np.zeros(k + 1, dtype=np.uint64)
    cof = np.zeros(max(k, 1), dtype=np.uint32)
    rc = _load().oracle_group(h.ctypes.data if n else None, n, lab.ctypes.data if n else None,
                              f.ctypes.data if k else None, k, order.ctypes.data, offsets.ctypes.data,
                              cof.ctypes.data)
    if rc != 0:
        raise OracleError(f"oracle_group returned {rc}")
    return order[:n].copy(), offsets, cof[:k].copy()


def centroids(feats) -> np.ndarray:
    f = np.ascontiguousarray(feats, dtype=FEAT_DTYPE)
    out = np.zeros((len(f), 2), dtype=np.float64)
    if len(f):
        _load().oracle_centroids(f.ctypes.data, len(f), out.ctypes.data)
    return out


class ComponentSampler:
    """One-component-at-a-time oracle for sampled parity at full size."""

    def __init__(self, hits, dt: int, width: int = 256, height: int = 256):
        self._h = _hits(hits)
        self._p = _load().oracle_index_new(self._h.ctypes.data, len(self._h), int(dt), width, height)
        if not self._p:
            raise OracleError("oracle_index_new failed")

    def component(self, seed: int, want_members: bool = False):
        L = _load()
        f = np.zeros(1, dtype=FEAT_DTYPE)
        cap = 1 << 16 if want_members else 0
        mem = np.zeros(max(cap, 1), dtype=np.uint32)
        m = L.oracle_index_component(self._p, int(seed), mem.ctypes.data if cap else None, cap, f.ctypes.data)
        if m < 0:
            raise OracleError("oracle_index_component failed")
        if want_members:
            if m > cap:
                raise OracleError("component larger than member buffer")
            return f[0], np.sort(mem[:m])
        return f[0]

    def close(self):
        if self._p:
            _load().oracle_index_delete(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
