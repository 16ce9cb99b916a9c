"""ToA-sharded multi-GPU clustering: binding of ``tpx_cluster_run_sharded``.

The whole protocol -- ranges, halo selection and exchange, boundary pairs,
union, relabelling, partial records and their fold -- runs inside the C-ABI
library (``csrc/sharded.cuh``, ``csrc/comm.cu``); this module only creates
communicators and marshals arguments (§3.2.3
l.117-119 temporal splitting, §4 l.173 border stitching).

Communicators (``tpx_comm``):
  * :class:`NcclComm` -- the product path: a library-owned NCCL communicator
    (one process per GPU, NVLink / NVSwitch), bootstrapped over a
    torch.distributed process group (rank 0's ``tpx_nccl_unique_id`` is
    broadcast, every rank calls ``tpx_nccl_comm_init``).
  * :class:`HostComm` -- host-callback transport for functional runs where
    NCCL cannot be used (in-process virtual ranks: :class:`ThreadAdapter`;
    gloo process groups, e.g. several ranks sharing one GPU:
    :class:`TorchAdapter`).  The library stages device buffers through
    pinned host memory and calls back into these adapters.
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import paper_2412_11809_b200 as _tpx

HIT_BYTES = 16
FEAT_BYTES = 64


class ShardError(RuntimeError):
    pass


# ------------------------------------------------------------ communicators
class _Comm:
    _h = None

    @property
    def handle(self):
        return self._h

    def rank_world(self):
        r, w = ctypes.c_int(0), ctypes.c_int(0)
        _tpx._check(_tpx._comm_rank(self._h, ctypes.byref(r), ctypes.byref(w)), "tpx_comm_rank")
        return r.value, w.value

    def close(self):
        if self._h:
            _tpx._comm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """128-byte NCCL bootstrap id (``tpx_nccl_unique_id``), created on rank 0."""
    uid = ctypes.create_string_buffer(128)
    _tpx._check(_tpx._nccl_unique_id(uid), "tpx_nccl_unique_id")
    return uid.raw


class NcclComm(_Comm):
    """Library-owned NCCL communicator on the current CUDA device.

    ``NcclComm()`` bootstraps over the default torch.distributed process group
    (or ``group``): rank 0's unique id is broadcast, every rank calls
    ``tpx_nccl_comm_init``.  ``NcclComm(rank=r, world=w, uid=...)`` takes an id
    distributed by other means (``world=1`` needs none)."""

    def __init__(self, group=None, rank: int | None = None, world: int | None = None, uid: bytes | None = None):
        if rank is None:
            import torch.distributed as dist

            rank, world = dist.get_rank(group), dist.get_world_size(group)
            obj = [nccl_unique_id() if rank == 0 else None]
            src = dist.get_global_rank(group, 0) if group is not None else 0
            dist.broadcast_object_list(obj, src=src, group=group)
            uid = obj[0]
        elif uid is None:
            if world != 1:
                raise ShardError("NcclComm(rank, world): a unique id is needed for world > 1")
            uid = nccl_unique_id()
        h = _tpx._vp()
        _tpx._check(_tpx._nccl_comm_init(int(rank), int(world), uid, ctypes.byref(h)), "tpx_nccl_comm_init")
        self._h = h


class HostComm(_Comm):
    """Host-callback transport around an adapter with ``rank``, ``world``,
    ``allgather(data: bytes) -> list[bytes]`` (rank order) and
    ``sendrecv(to, data, frm, nbytes) -> bytes`` (-1 = no peer)."""

    def __init__(self, adapter):
        self.adapter = adapter

        def allgather(_user, send, recv, nbytes):
            try:
                parts = adapter.allgather(ctypes.string_at(send, nbytes) if nbytes else b"")
                buf = b"".join(parts)
                ctypes.memmove(recv, buf, len(buf))
                return 0
            except Exception:  # surfaced to the library as a transport error
                return 1

        def sendrecv(_user, to, send, send_bytes, frm, recv, recv_bytes):
            try:
                data = ctypes.string_at(send, send_bytes) if (to >= 0 and send_bytes) else b""
                got = adapter.sendrecv(to, data, frm, recv_bytes)
                if frm >= 0 and recv_bytes:
                    ctypes.memmove(recv, got, recv_bytes)
                return 0
            except Exception:
                return 1

        # keep the callback objects alive as long as the communicator
        self._cb = (_tpx.ALLGATHER_FN(allgather), _tpx.SENDRECV_FN(sendrecv))
        h = _tpx._vp()
        _tpx._check(_tpx._comm_create_host(adapter.rank, adapter.world, self._cb[0], self._cb[1], None,
                                           ctypes.byref(h)), "tpx_comm_create_host")
        self._h = h

    def selftest(self, nbytes: int = 4096) -> int:
        return _tpx._comm_selftest(self._h, nbytes)


class ThreadGroup:
    """N virtual ranks as threads of one process (shared slots + barrier)."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.mail = {}
        self.lock = threading.Lock()


class ThreadAdapter:
    def __init__(self, group: ThreadGroup, rank: int):
        self.g, self.rank, self.world = group, rank, group.world

    def allgather(self, data: bytes):
        self.g.barrier.wait()
        self.g.slots[self.rank] = data
        self.g.barrier.wait()
        out = list(self.g.slots)
        self.g.barrier.wait()
        return out

    def sendrecv(self, to, data, frm, nbytes):
        if to >= 0:
            with self.g.lock:
                self.g.mail[(self.rank, to)] = data
        self.g.barrier.wait()
        got = b""
        if frm >= 0:
            with self.g.lock:
                got = self.g.mail.pop((frm, self.rank))
        self.g.barrier.wait()
        return got


class TorchAdapter:
    """torch.distributed on CPU tensors (gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def allgather(self, data: bytes):
        t = self.torch.frombuffer(bytearray(data), dtype=self.torch.uint8) if data else \
            self.torch.empty(0, dtype=self.torch.uint8)
        out = [self.torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return [o.numpy().tobytes() for o in out]

    def sendrecv(self, to, data, frm, nbytes):
        torch, dist = self.torch, self.dist
        ops = []
        if to >= 0 and data:
            ops.append(dist.P2POp(dist.isend, torch.frombuffer(bytearray(data), dtype=torch.uint8), self._peer(to),
                                  self.group))
        rbuf = torch.empty(nbytes if frm >= 0 else 0, dtype=torch.uint8)
        if frm >= 0 and nbytes:
            ops.append(dist.P2POp(dist.irecv, rbuf, self._peer(frm), self.group))
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return rbuf.numpy().tobytes()


# ------------------------------------------------------------------ the run
@dataclass
class ShardResult:
    labels: object      # this rank's labels (global input indices), n_r (int32 view of u32)
    features: object    # records whose label falls in this rank's block, ascending (uint8 [k, 64])
    n_clusters: int
    offset: int         # o_r, first global index of this rank's block
    stats: dict


class ShardedClusterer:
    """One context + workspace for ``tpx_cluster_run_sharded`` on ``comm``."""

    def __init__(self, dt_max: int, comm: _Comm, width: int = 256, height: int = 256):
        self.ctx = _tpx.Clusterer(dt_max, width, height)
        self.comm = comm
        self._ws = None

    def workspace_bytes(self, n: int) -> int:
        _, world = self.comm.rank_world()
        b = ctypes.c_size_t(0)
        _tpx._check(_tpx._sharded_ws(self.ctx._h, int(n), world, ctypes.byref(b)),
                    "tpx_cluster_sharded_workspace_bytes")
        return b.value

    def run(self, hits, n: int | None = None, labels=None, features=None, capacity: int | None = None,
            stream=None) -> ShardResult:
        import torch

        assert hits.is_cuda and hits.is_contiguous()
        if n is None:
            n = hits.numel() * hits.element_size() // HIT_BYTES
        dev = hits.device
        if labels is None:
            labels = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
        if capacity is None:
            capacity = n if features is None else features.numel() * features.element_size() // FEAT_BYTES
        if features is None:
            features = torch.empty((max(capacity, 1), FEAT_BYTES), dtype=torch.uint8, device=dev)
        need = self.workspace_bytes(n)
        if self._ws is None or self._ws.numel() < need or self._ws.device != dev:
            self._ws = None
            self._ws = torch.empty(need, dtype=torch.uint8, device=dev)
        k, off = _tpx._u64(0), _tpx._u64(0)
        rc = _tpx._run_sharded(self.ctx._h, self.comm.handle, hits.data_ptr(), int(n), labels.data_ptr(),
                               features.data_ptr(), int(capacity), ctypes.byref(k), ctypes.byref(off),
                               self._ws.data_ptr(), self._ws.numel(), _tpx._stream_handle(stream))
        if rc != _tpx.TPX_OK:
            raise ShardError(f"tpx_cluster_run_sharded: {_tpx.status_string(rc)} ({rc})")
        st = self.ctx.stats()
        return ShardResult(labels[:n], features[: min(k.value, capacity)], k.value, off.value, st)

    def close(self):
        self.ctx.close()
        self._ws = None


def cluster_sharded(hits, dt_max: int, comm: _Comm, width: int = 256, height: int = 256, stream=None) -> ShardResult:
    """One sharded run of this rank's block ``hits`` (device, [n_r, 16] bytes)."""
    c = ShardedClusterer(dt_max, comm, width, height)
    try:
        return c.run(hits, stream=stream)
    finally:
        c.close()
