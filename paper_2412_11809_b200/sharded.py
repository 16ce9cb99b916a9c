"""ToA-sharded multi-GPU clustering (§3.2.3 l.117-119).

One process (or, for tests, one thread) per GPU.  Rank r owns the
contiguous input-index block [o_r, o_r + n_r) of the t-ordered stream.  The
protocol (every compute step is a device kernel behind the C ABI, ``ops``;
every exchange is a collective on ``comm``):

  1. all-gather block sizes -> offsets; all-gather [minToA, maxToA] and check
     that no edge can skip a rank (minToA(r+2) > maxToA(r) + dt_max);
  2. rank r+1 selects its hits with toa <= maxToA(r) + dt_max (the forward
     halo of rank r) and sends them (and their block positions) to rank r;
  3. each rank clusters [owned | halo] with ``run_partial`` (features only
     from owned hits), translates labels to global input indices;
  4. rank r+1 sends back its own labels of the hits it lent; the halo hits'
     two labels form boundary pairs; all ranks all-gather the pairs and run
     the same union pass (smallest label wins);
  5. relabel owned hits; records of merged clusters become partials, are
     all-gathered, and each owner folds those whose final label it owns.

Concatenating the ranks' labels and records in rank order gives exactly the
single-GPU result (tests/test_gpu_sharded.py checks this bit for bit).
"""
from __future__ import annotations

import threading
from dataclasses import dataclass

import numpy as np

HIT_BYTES = 16
FEAT_BYTES = 64


class ShardError(RuntimeError):
    pass


# ---------------------------------------------------------------- communicators
class TorchComm:
    """torch.distributed process group (NCCL on GPUs, gloo on CPU).

    ``staged=True`` routes device tensors through host memory for every
    collective -- a gloo process group on GPU ranks (functional runs of the
    multi-process path where NCCL is unavailable, e.g. several ranks sharing
    one GPU); the NVLink path is NCCL with staged=False."""

    def __init__(self, group=None, staged: bool = False):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.staged = staged
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def allgather(self, t):
        """All-gather equal-shape tensors -> list (rank order)."""
        src = t.contiguous().cpu() if self.staged else t.contiguous()
        out = [src.new_empty(src.shape) for _ in range(self.world)]
        self.dist.all_gather(out, src, group=self.group)
        return [o.to(t.device) for o in out] if self.staged else out

    def exchange(self, send_to, send_tensors, recv_from, recv_tensors):
        """Point-to-point: send a list to one peer, receive a list from another."""
        ops = []
        P2POp, isend, irecv = self.dist.P2POp, self.dist.isend, self.dist.irecv
        sends = [t.contiguous().cpu() if self.staged else t.contiguous() for t in send_tensors]
        recvs = [t.new_empty(t.shape, device="cpu") if self.staged else t for t in recv_tensors]
        if send_to is not None:
            ops += [P2POp(isend, t, send_to, self.group) for t in sends]
        if recv_from is not None:
            ops += [P2POp(irecv, t, recv_from, self.group) for t in recvs]
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()
        if self.staged and recv_from is not None:
            for dst, src in zip(recv_tensors, recvs):
                dst.copy_(src)

    def barrier(self):
        self.dist.barrier(group=self.group)


class ThreadGroup:
    """Shared state for ThreadComm: N virtual ranks as threads of one process."""

    def __init__(self, world: int):
        self.world = world
        self.barrier = threading.Barrier(world)
        self.slots = [None] * world
        self.mail = {}
        self.lock = threading.Lock()


class ThreadComm:
    """In-process communicator (virtual ranks as threads): same protocol, same
    kernels, collectives replaced by copies -- the multi-rank path on one GPU."""

    def __init__(self, group: ThreadGroup, rank: int, device=None):
        self.g, self.rank, self.world = group, rank, group.world
        self.device = device

    def allgather(self, t):
        import torch

        if t.is_cuda:
            torch.cuda.current_stream(t.device).synchronize()
        self.g.barrier.wait()
        self.g.slots[self.rank] = t.detach().clone()
        self.g.barrier.wait()
        out = [s.to(t.device) for s in self.g.slots]
        self.g.barrier.wait()
        return out

    def exchange(self, send_to, send_tensors, recv_from, recv_tensors):
        import torch

        if send_to is not None:
            for t in send_tensors:
                if t.is_cuda:
                    torch.cuda.current_stream(t.device).synchronize()
            with self.g.lock:
                self.g.mail[(self.rank, send_to)] = [t.detach().clone() for t in send_tensors]
        self.g.barrier.wait()
        if recv_from is not None:
            with self.g.lock:
                got = self.g.mail.pop((recv_from, self.rank))
            for dst, src in zip(recv_tensors, got):
                dst.copy_(src.to(dst.device))
        self.g.barrier.wait()

    def barrier(self):
        self.g.barrier.wait()


# ----------------------------------------------------------------------- ops
class CudaOps:
    """Compute steps as C-ABI kernel calls on CUDA tensors (the product path)."""

    def __init__(self, dt_max: int, width: int = 256, height: int = 256):
        import torch

        import paper_2412_11809_b200 as tpx

        self.torch, self.tpx = torch, tpx
        self.dt = int(dt_max)
        self.clusterer = tpx.Clusterer(dt_max, width, height)
        self.device = torch.device("cuda", torch.cuda.current_device())

    def _ws(self, nbytes):
        return self.torch.empty(max(int(nbytes), 256), dtype=self.torch.uint8, device=self.device)

    def _u64(self, n=1):
        return self.torch.zeros(n, dtype=self.torch.int64, device=self.device)

    def toa_range(self, hits, n):
        mm = self._u64(2)
        self.tpx._check(self.tpx._shard_toa_range(hits.data_ptr() if n else None, n, mm.data_ptr(),
                                                  self.tpx._stream_handle(None)), "tpx_shard_toa_range")
        return mm

    def select_halo(self, hits, n, toa_limit):
        tpx = self.tpx
        ws = self._ws(tpx._size_query(tpx._shard_select_ws, n))
        halo = self.torch.empty((max(n, 1), HIT_BYTES), dtype=self.torch.uint8, device=self.device)
        idx = self.torch.empty(max(n, 1), dtype=self.torch.int32, device=self.device)
        cnt = self._u64()
        tpx._check(tpx._shard_select(hits.data_ptr() if n else None, n, int(toa_limit), halo.data_ptr(),
                                     idx.data_ptr(), cnt.data_ptr(), ws.data_ptr(), ws.numel(),
                                     tpx._stream_handle(None)), "tpx_shard_select_halo")
        c = int(cnt.item())
        return halo[:c].contiguous(), idx[:c].contiguous(), c

    def cluster_partial(self, hits, n, n_owned):
        labels, feats, k = self.clusterer.run_partial(hits, n, n_owned)
        return labels, feats, k

    def translate(self, labels, n, n_owned, own_off, halo_idx, next_off):
        tpx = self.tpx
        tpx._check(tpx._shard_translate(labels.data_ptr(), n, n_owned, own_off,
                                        halo_idx.data_ptr() if halo_idx.numel() else None, next_off,
                                        tpx._stream_handle(None)), "tpx_shard_translate_labels")

    def offset_feature_labels(self, feats, k, off):
        tpx = self.tpx
        tpx._check(tpx._shard_offset(feats.data_ptr() if k else None, k, int(off), tpx._stream_handle(None)),
                   "tpx_shard_offset_labels")

    def gather(self, labels, idx, c):
        out = self.torch.empty(max(c, 1), dtype=self.torch.int32, device=self.device)
        tpx = self.tpx
        tpx._check(tpx._shard_gather(labels.data_ptr(), idx.data_ptr() if c else None, c, out.data_ptr(),
                                     tpx._stream_handle(None)), "tpx_shard_gather_labels")
        return out[:c]

    def make_pairs(self, a, b, c):
        pairs = self.torch.empty((max(c, 1), 2), dtype=self.torch.int32, device=self.device)
        cnt = self._u64()
        tpx = self.tpx
        tpx._check(tpx._shard_pairs(a.data_ptr() if c else None, b.data_ptr() if c else None, c, pairs.data_ptr(),
                                    cnt.data_ptr(), tpx._stream_handle(None)), "tpx_shard_make_pairs")
        p = int(cnt.item())
        return pairs[:p].contiguous(), p

    def union_pairs(self, pairs, p):
        tpx = self.tpx
        ws = self._ws(tpx._size_query(tpx._shard_union_ws, p))
        keys = self.torch.empty(max(2 * p, 1), dtype=self.torch.int32, device=self.device)
        vals = self.torch.empty_like(keys)
        nmap = self._u64()
        tpx._check(tpx._shard_union(pairs.data_ptr() if p else None, p, keys.data_ptr(), vals.data_ptr(),
                                    nmap.data_ptr(), ws.data_ptr(), ws.numel(), tpx._stream_handle(None)),
                   "tpx_shard_union_pairs")
        return keys, vals, nmap

    def relabel(self, labels, n, mp):
        keys, vals, nmap = mp
        tpx = self.tpx
        tpx._check(tpx._shard_relabel(labels.data_ptr(), n, keys.data_ptr(), vals.data_ptr(), nmap.data_ptr(),
                                      tpx._stream_handle(None)), "tpx_shard_relabel")

    def split(self, feats, k, mp):
        keys, vals, nmap = mp
        tpx, torch = self.tpx, self.torch
        ws = self._ws(tpx._size_query(tpx._shard_split_ws, k))
        kept = torch.empty((max(k, 1), FEAT_BYTES), dtype=torch.uint8, device=self.device)
        part = torch.empty_like(kept)
        nk, npart = self._u64(), self._u64()
        tpx._check(tpx._shard_split(feats.data_ptr() if k else None, k, keys.data_ptr(), vals.data_ptr(),
                                    nmap.data_ptr(), kept.data_ptr(), nk.data_ptr(), part.data_ptr(),
                                    npart.data_ptr(), ws.data_ptr(), ws.numel(), tpx._stream_handle(None)),
                   "tpx_shard_split_features")
        a, b = int(nk.item()), int(npart.item())
        return kept[:a], a, part[:b].contiguous(), b

    def fold(self, kept, nk, partials, q, lo, hi, capacity):
        tpx, torch = self.tpx, self.torch
        ws = self._ws(tpx._size_query(tpx._shard_fold_ws, q))
        out = torch.empty((max(capacity, 1), FEAT_BYTES), dtype=torch.uint8, device=self.device)
        import ctypes

        n_out = ctypes.c_uint64(0)
        tpx._check(tpx._shard_fold(kept.data_ptr() if nk else None, nk, partials.data_ptr() if q else None, q,
                                   int(lo), int(hi), out.data_ptr(), capacity, ctypes.byref(n_out), ws.data_ptr(),
                                   ws.numel(), tpx._stream_handle(None)), "tpx_shard_fold_features")
        return out[: n_out.value], n_out.value

    # generic tensor helpers (device memory plumbing)
    def empty_hits(self, n):
        return self.torch.empty((max(n, 1), HIT_BYTES), dtype=self.torch.uint8, device=self.device)[:n]

    def empty_u32(self, n):
        return self.torch.empty(max(n, 1), dtype=self.torch.int32, device=self.device)[:n]

    def empty_feats(self, n):
        return self.torch.empty((max(n, 1), FEAT_BYTES), dtype=self.torch.uint8, device=self.device)[:n]

    def cat(self, a, b):
        return self.torch.cat([a.reshape(-1), b.reshape(-1)]).view(-1, a.shape[-1]) if a.dim() > 1 else \
            self.torch.cat([a, b])

    def scalar_tensor(self, values):
        return self.torch.tensor(values, dtype=self.torch.int64, device=self.device)

    def zeros_pairs(self, n):
        return self.torch.zeros((n, 2), dtype=self.torch.int32, device=self.device)

    def concat_rows(self, parts):
        return self.torch.cat(parts).contiguous()


# ------------------------------------------------------------------ protocol
@dataclass
class ShardResult:
    labels: object        # this rank's labels (global input indices), n_r
    features: object      # records whose label falls in this rank's block, ascending
    n_clusters: int
    offset: int
    stats: dict


def cluster_sharded(hits, dt_max: int, comm, ops) -> ShardResult:
    """Run the sharded protocol for this rank's block ``hits`` ([n_r, 16] bytes)."""
    G, r = comm.world, comm.rank
    n = int(hits.shape[0]) if hits.dim() > 1 else int(hits.numel() // HIT_BYTES)
    hits = hits.reshape(n, HIT_BYTES) if n else hits
    sizes = [int(t[0].item()) for t in comm.allgather(ops.scalar_tensor([n]))]
    if min(sizes) == 0:
        raise ShardError("every rank needs at least one hit")
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if offs[-1] >= 2**31:
        raise ShardError("sharded path supports < 2^31 hits in total")
    o_r = int(offs[r])
    mm = [tuple(int(v) for v in t.tolist()) for t in comm.allgather(ops.toa_range(hits, n))]
    for s in range(G):
        for t in range(s + 2, G):
            if mm[t][0] <= mm[s][1] + dt_max:
                raise ShardError(f"an edge could skip a rank ({s} -> {t}): blocks too small for dt_max")
    # 2. halo for rank r-1, exchange with neighbours
    if r > 0:
        halo_send, idx_send, c_send = ops.select_halo(hits, n, mm[r - 1][1] + dt_max)
    else:
        halo_send, idx_send, c_send = ops.empty_hits(0), ops.empty_u32(0), 0
    counts = [int(t[0].item()) for t in comm.allgather(ops.scalar_tensor([c_send]))]
    c_recv = counts[r + 1] if r + 1 < G else 0
    halo_recv, idx_recv = ops.empty_hits(c_recv), ops.empty_u32(c_recv)
    comm.exchange(r - 1 if r > 0 and c_send else None, [halo_send, idx_send],
                  r + 1 if c_recv else None, [halo_recv, idx_recv])
    # 3. cluster [owned | halo], features from owned hits only
    X = ops.cat(hits, halo_recv) if c_recv else hits
    labels, feats, k = ops.cluster_partial(X, n + c_recv, n)
    ops.translate(labels, n + c_recv, n, o_r, idx_recv, int(offs[r + 1]) if r + 1 < G else 0)
    ops.offset_feature_labels(feats, k, o_r)
    # 4. boundary pairs: my label vs the next rank's label of each halo hit
    lab_send = ops.gather(labels, idx_send, c_send) if c_send else ops.empty_u32(0)
    lab_peer = ops.empty_u32(c_recv)
    comm.exchange(r - 1 if r > 0 and c_send else None, [lab_send], r + 1 if c_recv else None, [lab_peer])
    pairs, p = ops.make_pairs(labels[n:n + c_recv], lab_peer, c_recv)
    pcounts = [int(t[0].item()) for t in comm.allgather(ops.scalar_tensor([p]))]
    pmax = max(pcounts)
    all_pairs, P = None, sum(pcounts)
    if P:
        pad = ops.zeros_pairs(pmax)
        pad[:p] = pairs[:p]
        gathered = comm.allgather(pad)
        all_pairs = ops.concat_rows([g[:c] for g, c in zip(gathered, pcounts)])
    mp = ops.union_pairs(all_pairs, P) if P else ops.union_pairs(None, 0)
    # 5. relabel, split records, gather partials, fold the ones this rank owns
    ops.relabel(labels, n, mp)
    kept, nk, part, q = ops.split(feats, k, mp)
    qcounts = [int(t[0].item()) for t in comm.allgather(ops.scalar_tensor([q]))]
    Q = sum(qcounts)
    all_part = ops.empty_feats(0)
    if Q:
        qmax = max(qcounts)
        padf = ops.empty_feats(qmax)
        padf[:q] = part[:q]
        gathered = comm.allgather(padf)
        all_part = ops.concat_rows([g[:c] for g, c in zip(gathered, qcounts)])
    out, k_out = ops.fold(kept, nk, all_part, Q, o_r, o_r + n, nk + Q)
    stats = {"halo_sent": c_send, "halo_recv": c_recv, "pairs": p, "pairs_total": P, "partials": q,
             "partials_total": Q, "local_clusters": k}
    return ShardResult(labels[:n], out, k_out, o_r, stats)
