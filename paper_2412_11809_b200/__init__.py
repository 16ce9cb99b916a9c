"""B200-native Timepix3 hit clustering (arXiv 2412.11809 hot path).

Thin Python binding over the C-ABI library ``lib/libtpxcluster.so``
(``include/tpx_cluster.h``): argument marshalling only.  Every step of the
path -- ToA sort, windowed neighbour search, union-find, canonical labels,
compaction, feature reductions, centroids -- runs in the library's sm_100a
kernels.  PyTorch supplies device memory and streams.  There is no CPU
fallback: if the library is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libtpxcluster.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(or python paper_2412_11809_b200/build.py); there is no CPU fallback")

_lib = ctypes.CDLL(LIB_PATH)

TPX_OK = 0
TPX_ERR_CAPACITY = -5
VARIANT_LOCAL, VARIANT_GLOBAL, VARIANT_STATIC = 0, 1, 2

#: 64-byte cluster feature record (tpx_cluster_features).
FEATURE_DTYPE = np.dtype(
    [("label", "<u4"), ("size", "<u4"), ("toa_min", "<u8"), ("toa_max", "<u8"),
     ("tot_sum", "<u8"), ("sum_x", "<u8"), ("sum_y", "<u8"), ("sum_tot_x", "<u8"),
     ("sum_tot_y", "<u8")]
)

_vp, _u64, _u32, _int = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int


class RunStats(ctypes.Structure):
    _fields_ = [
        ("n_hits", _u64), ("n_clusters", _u64), ("sort_path", _u32), ("sort_retries", _u32),
        ("cross_pairs", _u64), ("kernel_launches", _u32), ("n_stages", _u32),
        ("stage_ms", ctypes.c_float * 16),
        ("open_hits", _u64), ("overflow_hits", _u64), ("tile_phase_cycles", _u64 * 16),
        ("tile_dense", _u32), ("reserved0", _u32),
    ]


def _proto(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_abi_version = _proto("tpx_abi_version", _int)
_status_string = _proto("tpx_status_string", ctypes.c_char_p, _int)
_create = _proto("tpx_cluster_create", _int, _u64, _int, _u32, _u32, ctypes.POINTER(_vp))
_destroy = _proto("tpx_cluster_destroy", None, _vp)
_ws_bytes = _proto("tpx_cluster_workspace_bytes", _int, _vp, _u64, ctypes.POINTER(ctypes.c_size_t))
_run = _proto("tpx_cluster_run", _int, _vp, _vp, _u64, _vp, _vp, _u64, ctypes.POINTER(_u64), _vp,
              ctypes.c_size_t, _vp)
_host_ws_bytes = _proto("tpx_cluster_host_workspace_bytes", _int, _vp, _u64, _u64,
                        ctypes.POINTER(ctypes.c_size_t))
_run_host = _proto("tpx_cluster_run_host", _int, _vp, _vp, _u64, _vp, _vp, _u64, ctypes.POINTER(_u64), _vp,
                   ctypes.c_size_t, _vp)
_centroids = _proto("tpx_cluster_centroids", _int, _vp, _u64, _vp, _vp)
_last_stats = _proto("tpx_cluster_last_stats", _int, _vp, ctypes.POINTER(RunStats))
_set_profiling = _proto("tpx_cluster_set_profiling", _int, _vp, _int)
_set_tile_mode = _proto("tpx_cluster_set_tile_mode", _int, _vp, _int)
TILE_MODES = {"auto": 0, "sparse": 1, "dense": 2, "cell": 4}
_stage_name = _proto("tpx_cluster_stage_name", ctypes.c_char_p, _int)
_run_partial = _proto("tpx_cluster_run_partial", _int, _vp, _vp, _u64, _u64, _vp, _vp, _u64, ctypes.POINTER(_u64),
                      _vp, ctypes.c_size_t, _vp)
_size_t_p = ctypes.POINTER(ctypes.c_size_t)
_run_grouped = _proto("tpx_cluster_run_grouped", _int, _vp, _vp, _u64, _vp, _vp, _vp, _u64, ctypes.POINTER(_u64),
                      _vp, _vp, _vp, _vp, ctypes.c_size_t, _vp)
# host-buffer pipeline (include/tpx_cluster.h, "Host-buffer pipeline")
_pipe_ws = _proto("tpx_pipeline_workspace_bytes", _int, _vp, _u64, _u64, _int, _size_t_p)
_pipe_create = _proto("tpx_pipeline_create", _int, _u64, _int, _u32, _u32, _u64, _u64, _int, _vp, ctypes.c_size_t,
                      ctypes.POINTER(_vp))
_pipe_submit = _proto("tpx_pipeline_submit", _int, _vp, _vp, _u64, _vp, _vp, _u64, ctypes.POINTER(_u64))
_pipe_wait = _proto("tpx_pipeline_wait", _int, _vp, _u64, ctypes.POINTER(_u64))
_pipe_mark = _proto("tpx_pipeline_mark", _int, _vp, _int)
_pipe_elapsed = _proto("tpx_pipeline_elapsed_ms", _int, _vp, ctypes.POINTER(ctypes.c_float))
_pipe_destroy = _proto("tpx_pipeline_destroy", None, _vp)
# ToA-sharded run + communicators (include/tpx_cluster.h, "ToA-sharded multi-GPU clustering")
ALLGATHER_FN = ctypes.CFUNCTYPE(_int, _vp, _vp, _vp, ctypes.c_size_t)
SENDRECV_FN = ctypes.CFUNCTYPE(_int, _vp, _int, _vp, ctypes.c_size_t, _int, _vp, ctypes.c_size_t)
_nccl_unique_id = _proto("tpx_nccl_unique_id", _int, ctypes.c_char_p)
_nccl_comm_init = _proto("tpx_nccl_comm_init", _int, _int, _int, ctypes.c_char_p, ctypes.POINTER(_vp))
_comm_create_host = _proto("tpx_comm_create_host", _int, _int, _int, ALLGATHER_FN, SENDRECV_FN, _vp,
                           ctypes.POINTER(_vp))
_comm_destroy = _proto("tpx_comm_destroy", None, _vp)
_comm_rank = _proto("tpx_comm_rank", _int, _vp, ctypes.POINTER(_int), ctypes.POINTER(_int))
_comm_selftest = _proto("tpx_comm_selftest", _int, _vp, ctypes.c_size_t)
_sharded_ws = _proto("tpx_cluster_sharded_workspace_bytes", _int, _vp, _u64, _int, _size_t_p)
_run_sharded = _proto("tpx_cluster_run_sharded", _int, _vp, _vp, _vp, _u64, _vp, _vp, _u64, ctypes.POINTER(_u64),
                      ctypes.POINTER(_u64), _vp, ctypes.c_size_t, _vp)

ABI_VERSION = _abi_version()


class TpxError(RuntimeError):
    def __init__(self, status: int, what: str = ""):
        self.status = status
        super().__init__(f"{what}: {status_string(status)} ({status})")


def _check(rc: int, what: str):
    if rc != TPX_OK:
        raise TpxError(rc, what)


def _size_query(fn, n: int) -> int:
    b = ctypes.c_size_t(0)
    _check(fn(int(n), ctypes.byref(b)), fn.__name__)
    return b.value


def status_string(status: int) -> str:
    return _status_string(status).decode()


def stage_name(i: int) -> str:
    return _stage_name(i).decode()


def _torch():
    import torch  # plumbing only: device memory + streams

    return torch


def _stream_handle(stream) -> int:
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


class Clusterer:
    """One library context (``tpx_cluster_create``); not thread-safe.

    ``dt_max`` is in ToA ticks (1.5625 ns).  ``run`` takes a CUDA tensor of
    n 16-byte ``tpx_hit`` records and returns ``(labels, features, n_clusters)``
    as CUDA tensors (labels: int32 view of u32; features: uint8 [k, 64]).
    """

    def __init__(self, dt_max: int, width: int = 256, height: int = 256, variant: int = VARIANT_LOCAL):
        h = _vp()
        rc = _create(int(dt_max), int(variant), int(width), int(height), ctypes.byref(h))
        if rc != TPX_OK:
            raise TpxError(rc, "tpx_cluster_create")
        self._h = h
        self.dt_max, self.width, self.height = int(dt_max), int(width), int(height)
        self._ws = None

    # -- resources ---------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            _destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def workspace_bytes(self, n: int) -> int:
        b = ctypes.c_size_t(0)
        rc = _ws_bytes(self._h, int(n), ctypes.byref(b))
        if rc != TPX_OK:
            raise TpxError(rc, "tpx_cluster_workspace_bytes")
        return b.value

    def host_workspace_bytes(self, n: int, capacity: int) -> int:
        b = ctypes.c_size_t(0)
        rc = _host_ws_bytes(self._h, int(n), int(capacity), ctypes.byref(b))
        if rc != TPX_OK:
            raise TpxError(rc, "tpx_cluster_host_workspace_bytes")
        return b.value

    def _workspace(self, nbytes: int, device):
        torch = _torch()
        device = torch.device(device)
        if device.type == "cuda" and device.index is None:  # "cuda" -> "cuda:<current>" (cache key)
            device = torch.device("cuda", torch.cuda.current_device())
        if self._ws is None or self._ws.numel() < nbytes or self._ws.device != device:
            self._ws = None
            self._ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self._ws

    def set_profiling(self, on: bool | int = True):
        """False/0 off, True/1 stage events, 2 stage events + tile phase clocks."""
        _check(_set_profiling(self._h, int(on)), "tpx_cluster_set_profiling")

    def set_tile_mode(self, mode: str = "auto"):
        """'auto' (density probe), 'sparse' (k_tile_csr), 'dense' (k_tile_cc) or
        'cell' (k_tile_cell) tile configuration."""
        _check(_set_tile_mode(self._h, TILE_MODES[mode]), "tpx_cluster_set_tile_mode")

    def stats(self) -> dict:
        s = RunStats()
        _last_stats(self._h, ctypes.byref(s))
        d = {k: getattr(s, k) for k, _ in RunStats._fields_ if k not in ("stage_ms", "tile_phase_cycles")}
        d["stage_ms"] = {stage_name(i): s.stage_ms[i] for i in range(s.n_stages)}
        d["tile_phase_cycles"] = list(s.tile_phase_cycles)
        return d

    # -- the hot path ------------------------------------------------------
    def run(self, hits, n: int | None = None, labels=None, features=None, capacity: int | None = None,
            workspace=None, stream=None, check: bool = True):
        """Cluster hits resident on the GPU (``tpx_cluster_run``)."""
        torch = _torch()
        assert hits.is_cuda and hits.is_contiguous()
        if n is None:
            n = hits.numel() * hits.element_size() // 16
        dev = hits.device
        if labels is None:
            labels = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        if capacity is None:
            capacity = n if features is None else features.numel() * features.element_size() // 64
        if features is None:
            features = torch.empty((max(capacity, 1), 64), dtype=torch.uint8, device=dev)
        if workspace is None:
            workspace = self._workspace(self.workspace_bytes(n), dev)
        k = _u64(0)
        rc = _run(self._h, hits.data_ptr(), int(n), labels.data_ptr(), features.data_ptr(), int(capacity),
                  ctypes.byref(k), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
                  _stream_handle(stream))
        if check and rc not in (TPX_OK,):
            raise TpxError(rc, "tpx_cluster_run")
        kk = min(k.value, capacity)
        return labels[:n], features[:kk], k.value

    def run_grouped(self, hits, n: int | None = None, shapes: bool = True, stream=None, out: dict | None = None,
                    workspace=None):
        """``tpx_cluster_run_grouped``: labels, features, optional shape records
        and the cluster-contiguous order (Alg. GPU Step 6).

        Returns ``(labels, features, shapes|None, order, offsets, cluster_of, k)``
        (device tensors; offsets has k + 1 entries).  ``out`` may hold
        preallocated tensors under those names (capacity n).
        """
        torch = _torch()
        assert hits.is_cuda and hits.is_contiguous()
        if n is None:
            n = hits.numel() * hits.element_size() // 16
        dev = hits.device
        cap = max(n, 1)
        o = out or {}
        labels = o.get("labels", None)
        if labels is None:
            labels = torch.empty(cap, dtype=torch.int32, device=dev)
        features = o.get("features", None)
        if features is None:
            features = torch.empty((cap, 64), dtype=torch.uint8, device=dev)
        shp = o.get("shapes", None)
        if shp is None and shapes:
            shp = torch.empty((cap, 32), dtype=torch.uint8, device=dev)
        order = o.get("order", None)
        if order is None:
            order = torch.empty(cap, dtype=torch.int32, device=dev)
        offsets = o.get("offsets", None)
        if offsets is None:
            offsets = torch.empty(cap + 1, dtype=torch.int32, device=dev)
        cluster_of = o.get("cluster_of", None)
        if cluster_of is None:
            cluster_of = torch.empty(cap, dtype=torch.int32, device=dev)
        if workspace is None:
            workspace = self._workspace(self.workspace_bytes(n), dev)
        k = _u64(0)
        rc = _run_grouped(self._h, hits.data_ptr(), int(n), labels.data_ptr(), features.data_ptr(),
                          shp.data_ptr() if shapes else None, int(cap), ctypes.byref(k), order.data_ptr(),
                          offsets.data_ptr(), cluster_of.data_ptr(), workspace.data_ptr(),
                          workspace.numel() * workspace.element_size(), _stream_handle(stream))
        _check(rc, "tpx_cluster_run_grouped")
        kk = k.value
        return (labels[:n], features[:kk], shp[:kk] if shapes else None, order[:n], offsets[: kk + 1],
                cluster_of[:kk], kk)

    def run_partial(self, hits, n: int, n_owned: int, stream=None):
        """``tpx_cluster_run_partial``: the first n_owned hits are owned, the rest
        a borrowed halo (features and records only from owned hits)."""
        torch = _torch()
        dev = hits.device
        labels = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        features = torch.empty((max(n_owned, 1), 64), dtype=torch.uint8, device=dev)
        workspace = self._workspace(self.workspace_bytes(n), dev)
        k = _u64(0)
        rc = _run_partial(self._h, hits.data_ptr(), int(n), int(n_owned), labels.data_ptr(), features.data_ptr(),
                          int(n_owned), ctypes.byref(k), workspace.data_ptr(), workspace.numel(),
                          _stream_handle(stream))
        _check(rc, "tpx_cluster_run_partial")
        return labels[:n], features[: k.value], k.value

    def run_host(self, hits_host, labels_host, features_host, capacity: int | None = None, workspace=None,
                 stream=None, check: bool = True) -> int:
        """End-to-end with HOST buffers (``tpx_cluster_run_host``).

        ``hits_host`` / ``labels_host`` / ``features_host`` are CPU tensors
        (pinned for asynchronous DMA) or numpy arrays; returns n_clusters.
        """
        def ptr(a):
            return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

        def nbytes(a):
            return a.numel() * a.element_size() if hasattr(a, "numel") else a.nbytes

        n = nbytes(hits_host) // 16
        if capacity is None:
            capacity = nbytes(features_host) // 64
        torch = _torch()
        if workspace is None:
            workspace = self._workspace(self.host_workspace_bytes(n, capacity), torch.device("cuda"))
        k = _u64(0)
        rc = _run_host(self._h, ptr(hits_host), int(n), ptr(labels_host), ptr(features_host), int(capacity),
                       ctypes.byref(k), workspace.data_ptr(), workspace.numel(), _stream_handle(stream))
        if check and rc != TPX_OK:
            raise TpxError(rc, "tpx_cluster_run_host")
        return k.value


class StreamConfig(ctypes.Structure):
    _fields_ = [("dt_max_ticks", _u64), ("width", _u32), ("height", _u32), ("buffer_hits", _u64),
                ("reserve_hits", _u64), ("disorder_ticks", _u64), ("closing_ticks", _u64),
                ("max_device_hits", _u64)]


class StreamBatch(ctypes.Structure):
    _fields_ = [("seq", _u64), ("n_clusters", _u64), ("n_hits", _u64), ("clusters", _vp), ("hits", _vp),
                ("hit_index", _vp)]


class StreamStats(ctypes.Structure):
    _fields_ = [("hits_in", _u64), ("hits_out", _u64), ("clusters_out", _u64), ("buffers", _u64),
                ("carried_max", _u64), ("carried_last", _u64), ("late_hits", _u64), ("device_ms", ctypes.c_double)]


#: 80-byte tpx_stream_cluster record.
STREAM_CLUSTER_DTYPE = np.dtype(
    [("label", "<u8"), ("offset", "<u8"), ("size", "<u4"), ("reserved", "<u4"), ("toa_min", "<u8"),
     ("toa_max", "<u8"), ("tot_sum", "<u8"), ("sum_x", "<u8"), ("sum_y", "<u8"), ("sum_tot_x", "<u8"),
     ("sum_tot_y", "<u8")]
)
assert STREAM_CLUSTER_DTYPE.itemsize == 80
_HIT_DTYPE = np.dtype([("toa", "<u8"), ("x", "<u2"), ("y", "<u2"), ("tot", "<u2"), ("reserved", "<u2")])

_stream_ws = _proto("tpx_stream_workspace_bytes", _int, ctypes.POINTER(StreamConfig), _size_t_p)
_stream_create = _proto("tpx_stream_create", _int, ctypes.POINTER(StreamConfig), _vp, ctypes.c_size_t, _vp,
                        ctypes.POINTER(_vp))
_stream_push = _proto("tpx_stream_push", _int, _vp, _vp, _u64)
_stream_flush = _proto("tpx_stream_flush", _int, _vp)
_stream_pop = _proto("tpx_stream_pop", _int, _vp, ctypes.POINTER(StreamBatch))
_stream_stats = _proto("tpx_stream_get_stats", _int, _vp, ctypes.POINTER(StreamStats))
_stream_destroy = _proto("tpx_stream_destroy", None, _vp)
_stream_rh_ws = _proto("tpx_stream_run_host_workspace_bytes", _int, ctypes.POINTER(StreamConfig), _size_t_p)
_stream_rh = _proto("tpx_stream_run_host", _int, ctypes.POINTER(StreamConfig), _vp, _u64, _vp, _vp, _u64,
                    ctypes.POINTER(_u64), _vp, ctypes.c_size_t, _vp, ctypes.POINTER(StreamStats))
_buffill_assign = _proto("tpx_buffill_assign", _int, _vp, _u64, _u64, _u64, _u64, _u64, _vp, _vp, _u64,
                         ctypes.POINTER(_u64))


def buffill_assign(hits: np.ndarray, b: int, b_t: int, t: int, t_closing: int):
    """Host-only: buffer id per hit and the cut of each buffer, as the stream
    assigns them (Alg. "Hit buffer filling")."""
    h = np.ascontiguousarray(hits)
    n = len(h)
    ids = np.zeros(max(n, 1), dtype=np.uint32)
    cap = n + 2
    cuts = np.zeros(cap, dtype=np.uint64)
    nb = _u64(0)
    _check(_buffill_assign(h.ctypes.data if n else None, n, int(b), int(b_t), int(t), int(t_closing),
                           ids.ctypes.data, cuts.ctypes.data, cap, ctypes.byref(nb)), "tpx_buffill_assign")
    return ids[:n], [int(c) for c in cuts[: nb.value]]


class StreamRunner:
    """``tpx_stream_run_host``: one-shot host-to-host clustering of a whole
    stream in host memory (BufFill + exact carry, copy/compute overlap)."""

    def __init__(self, dt_max: int, buffer_hits: int, reserve_hits: int, disorder_ticks: int, closing_ticks: int,
                 max_device_hits: int | None = None, width: int = 256, height: int = 256):
        torch = _torch()
        self.cfg = StreamConfig(int(dt_max), int(width), int(height), int(buffer_hits), int(reserve_hits),
                                int(disorder_ticks), int(closing_ticks),
                                int(max_device_hits or 2 * (buffer_hits + reserve_hits)))
        b = ctypes.c_size_t(0)
        _check(_stream_rh_ws(ctypes.byref(self.cfg), ctypes.byref(b)), "tpx_stream_run_host_workspace_bytes")
        self._ws = torch.empty(max(b.value, 256), dtype=torch.uint8, device="cuda")
        self.last_stats = None

    @staticmethod
    def _ptr(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    def run(self, hits_host, order_out, clusters_out, capacity: int | None = None, stream=None) -> int:
        """hits_host: (pinned) CPU tensor / numpy array of n 16-byte hits;
        order_out: n u32; clusters_out: capacity x 80 bytes.  Returns k."""
        nb = hits_host.numel() * hits_host.element_size() if hasattr(hits_host, "numel") else hits_host.nbytes
        n = nb // 16
        if capacity is None:
            cb = clusters_out.numel() * clusters_out.element_size() if hasattr(clusters_out, "numel") \
                else clusters_out.nbytes
            capacity = cb // 80
        k = _u64(0)
        st = StreamStats()
        _check(_stream_rh(ctypes.byref(self.cfg), self._ptr(hits_host), int(n), self._ptr(order_out),
                          self._ptr(clusters_out), int(capacity), ctypes.byref(k), self._ws.data_ptr(),
                          self._ws.numel(), _stream_handle(stream), ctypes.byref(st)), "tpx_stream_run_host")
        self.last_stats = {f: getattr(st, f) for f, _ in StreamStats._fields_}
        return k.value


class Stream:
    """``tpx_stream_*``: push hits in readout order, pop batches of final
    clusters (labels = smallest arrival index; Step-6 order)."""

    def __init__(self, dt_max: int, buffer_hits: int, reserve_hits: int, disorder_ticks: int, closing_ticks: int,
                 max_device_hits: int | None = None, width: int = 256, height: int = 256, stream=None):
        torch = _torch()
        cfg = StreamConfig(int(dt_max), int(width), int(height), int(buffer_hits), int(reserve_hits),
                           int(disorder_ticks), int(closing_ticks),
                           int(max_device_hits or 2 * (buffer_hits + reserve_hits)))
        b = ctypes.c_size_t(0)
        _check(_stream_ws(ctypes.byref(cfg), ctypes.byref(b)), "tpx_stream_workspace_bytes")
        self._ws = torch.empty(max(b.value, 256), dtype=torch.uint8, device="cuda")
        h = _vp()
        _check(_stream_create(ctypes.byref(cfg), self._ws.data_ptr(), self._ws.numel(), _stream_handle(stream),
                              ctypes.byref(h)), "tpx_stream_create")
        self._h = h

    def push(self, hits: np.ndarray):
        h = np.ascontiguousarray(hits)
        assert h.dtype.itemsize == 16
        _check(_stream_push(self._h, h.ctypes.data if len(h) else None, len(h)), "tpx_stream_push")

    def flush(self):
        _check(_stream_flush(self._h), "tpx_stream_flush")

    def pop(self):
        """Next batch as numpy copies ``{seq, clusters, hits, hit_index}`` or None."""
        bt = StreamBatch()
        r = _stream_pop(self._h, ctypes.byref(bt))
        if r < 0:
            _check(r, "tpx_stream_pop")
        if r == 0:
            return None

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            buf = (ctypes.c_uint8 * (n * dt.itemsize)).from_address(ptr)
            return np.frombuffer(buf, dtype=dt).copy()

        return {"seq": bt.seq, "clusters": arr(bt.clusters, bt.n_clusters, STREAM_CLUSTER_DTYPE),
                "hits": arr(bt.hits, bt.n_hits, _HIT_DTYPE), "hit_index": arr(bt.hit_index, bt.n_hits,
                                                                             np.dtype("<u8"))}

    def stats(self) -> dict:
        st = StreamStats()
        _check(_stream_stats(self._h, ctypes.byref(st)), "tpx_stream_get_stats")
        return {k: getattr(st, k) for k, _ in StreamStats._fields_}

    def close(self):
        if getattr(self, "_h", None):
            _stream_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Pipeline:
    """``tpx_pipeline_*``: overlap host<->device copies of one buffer with the
    kernels of another (``depth`` slots, native worker threads).  Buffers are
    CPU tensors (pinned) or numpy arrays and must stay alive until ``wait``."""

    def __init__(self, dt_max: int, max_hits: int, capacity: int, depth: int = 2, width: int = 256,
                 height: int = 256, variant: int = VARIANT_LOCAL):
        torch = _torch()
        proto = Clusterer(dt_max, width, height, variant)
        b = ctypes.c_size_t(0)
        _check(_pipe_ws(proto._h, int(max_hits), int(capacity), int(depth), ctypes.byref(b)),
               "tpx_pipeline_workspace_bytes")
        proto.close()
        self._ws = torch.empty(max(b.value, 256), dtype=torch.uint8, device="cuda")
        h = _vp()
        _check(_pipe_create(int(dt_max), int(variant), int(width), int(height), int(max_hits), int(capacity),
                            int(depth), self._ws.data_ptr(), self._ws.numel(), ctypes.byref(h)), "tpx_pipeline_create")
        self._h = h
        self._keep = {}

    @staticmethod
    def _ptr(a):
        return a.data_ptr() if hasattr(a, "data_ptr") else a.ctypes.data

    @staticmethod
    def _nbytes(a):
        return a.numel() * a.element_size() if hasattr(a, "numel") else a.nbytes

    def submit(self, hits_host, labels_host, features_host, capacity: int | None = None) -> int:
        n = self._nbytes(hits_host) // 16
        if capacity is None:
            capacity = self._nbytes(features_host) // 64
        t = _u64(0)
        _check(_pipe_submit(self._h, self._ptr(hits_host), int(n), self._ptr(labels_host), self._ptr(features_host),
                            int(capacity), ctypes.byref(t)), "tpx_pipeline_submit")
        self._keep[t.value] = (hits_host, labels_host, features_host)
        return t.value

    def wait(self, ticket: int, check: bool = True) -> int:
        k = _u64(0)
        rc = _pipe_wait(self._h, int(ticket), ctypes.byref(k))
        self._keep.pop(ticket, None)
        if check:
            _check(rc, "tpx_pipeline_wait")
        return k.value

    def mark(self, which: int):
        _check(_pipe_mark(self._h, int(which)), "tpx_pipeline_mark")

    def elapsed_ms(self) -> float:
        ms = ctypes.c_float(0)
        _check(_pipe_elapsed(self._h, ctypes.byref(ms)), "tpx_pipeline_elapsed_ms")
        return ms.value

    def close(self):
        if getattr(self, "_h", None):
            _pipe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def centroids(features, stream=None):
    """fp64 ToT-weighted centroids [k, 2] of device feature records."""
    torch = _torch()
    k = features.numel() * features.element_size() // 64
    out = torch.empty((max(k, 1), 2), dtype=torch.float64, device=features.device)
    rc = _centroids(features.data_ptr(), int(k), out.data_ptr(), _stream_handle(stream))
    if rc != TPX_OK:
        raise TpxError(rc, "tpx_cluster_centroids")
    return out[:k]


SHAPE_DTYPE = np.dtype(
    [("x_min", "<u2"), ("x_max", "<u2"), ("y_min", "<u2"), ("y_max", "<u2"),
     ("sum_xx", "<u8"), ("sum_xy", "<u8"), ("sum_yy", "<u8")]
)


def shapes_to_numpy(t) -> np.ndarray:
    """A (k, 32) uint8 tensor of tpx_cluster_shape records -> structured array."""
    a = t.contiguous().cpu().numpy() if hasattr(t, "cpu") else np.asarray(t)
    return a.reshape(-1).view(SHAPE_DTYPE).copy()


def features_to_numpy(features) -> np.ndarray:
    """Device/host feature bytes -> structured numpy array (FEATURE_DTYPE)."""
    a = features.detach().cpu().contiguous().numpy() if hasattr(features, "detach") else np.asarray(features)
    return a.reshape(-1).view(np.uint8).view(FEATURE_DTYPE)
