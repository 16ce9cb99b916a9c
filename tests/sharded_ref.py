"""CPU model of the ToA-sharded protocol -- TEST INFRASTRUCTURE.

The product protocol runs inside the C-ABI library
(paper_2412_11809_b200/csrc/sharded.cuh, tpx_cluster_run_sharded).  This is
a plain Python/numpy model of the same exchange steps (halo selection,
halo send/recv, label pairs, union pass, relabel, partial records and their
fold, §3.2.3 l.117-119) that runs on CPU tensors
with a gloo process group or in-process threads, every per-rank compute step
done with numpy and the oracle.  tests/test_sharded_protocol.py checks that
the scheme itself is exact (concatenated outputs == oracle) at world size
2..5 on CPU; the native implementation is checked bit for bit on the GPU
(tests/test_gpu_sharded.py).
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from tests import pins
from tpxgen import HIT_DTYPE

import threading
from dataclasses import dataclass

HIT_BYTES = 16
FEAT_BYTES = 64


class ModelShardError(RuntimeError):
    pass


# ---- tensor communicators of the model (torch.distributed / in-process threads)
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



FEAT = oracle.FEAT_DTYPE


def _hits(t) -> np.ndarray:
    return t.contiguous().numpy().reshape(-1).view(np.uint8).view(HIT_DTYPE)


def _feats_tensor(f: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(f).view(np.uint8).reshape(-1, 64).copy())


def _feats(t) -> np.ndarray:
    return t.contiguous().numpy().reshape(-1).view(FEAT)


class NumpyOps:
    def __init__(self, dt_max: int, width: int = 256, height: int = 256):
        self.dt, self.w, self.h = int(dt_max), width, height

    # plumbing
    def scalar_tensor(self, values):
        return torch.tensor(values, dtype=torch.int64)

    def empty_hits(self, n):
        return torch.zeros((n, 16), dtype=torch.uint8)

    def empty_u32(self, n):
        return torch.zeros(n, dtype=torch.int32)

    def empty_feats(self, n):
        return torch.zeros((n, 64), dtype=torch.uint8)

    def zeros_pairs(self, n):
        return torch.zeros((n, 2), dtype=torch.int32)

    def cat(self, a, b):
        return torch.cat([a, b])

    def concat_rows(self, parts):
        return torch.cat(parts).contiguous()

    # compute steps
    def toa_range(self, hits, n):
        t = _hits(hits)["toa"].astype(np.int64)
        return torch.tensor([t.min(), t.max()], dtype=torch.int64)

    def select_halo(self, hits, n, limit):
        h = _hits(hits)
        idx = np.nonzero(h["toa"] <= np.uint64(limit))[0]
        return hits[torch.from_numpy(idx)].contiguous(), torch.from_numpy(idx.astype(np.int32)), len(idx)

    def cluster_partial(self, X, n, n_owned):
        h = _hits(X)
        labels, _ = oracle.cluster(h, self.dt, self.w, self.h)
        own = labels[:n_owned]
        f = pins.features_from_labels(h[:n_owned], own)
        rec = np.zeros(len(f["label"]), dtype=FEAT)
        for k in pins.FEAT_FIELDS:
            rec[k] = f[k]
        return torch.from_numpy(labels.astype(np.int64).astype(np.int32)), _feats_tensor(rec), len(rec)

    def translate(self, labels, n, n_owned, own_off, halo_idx, next_off):
        L = labels.numpy().view(np.uint32).astype(np.int64)
        hi = halo_idx.numpy().view(np.uint32).astype(np.int64)
        out = np.where(L < n_owned, own_off + L, next_off + hi[np.clip(L - n_owned, 0, max(len(hi) - 1, 0))]
                       if len(hi) else own_off + L)
        labels.copy_(torch.from_numpy(out.astype(np.uint32).view(np.int32)))

    def offset_feature_labels(self, feats, k, off):
        if k:
            f = _feats(feats[:k]).copy()
            f["label"] += np.uint32(off)
            feats[:k] = _feats_tensor(f)

    def gather(self, labels, idx, c):
        return labels[idx.long()].clone()

    def make_pairs(self, a, b, c):
        keep = (a != b).nonzero().flatten()
        p = torch.stack([a[keep], b[keep]], 1).to(torch.int32).contiguous()
        return p, len(keep)

    def union_pairs(self, pairs, P):
        if not P:
            return {}
        pr = pairs.numpy().view(np.uint32).reshape(-1, 2).astype(np.int64)
        parent = {}

        def find(x):
            parent.setdefault(x, x)
            while parent[x] != x:
                parent[x] = parent[parent[x]]
                x = parent[x]
            return x

        for a, b in pr.tolist():
            ra, rb = find(a), find(b)
            if ra != rb:
                parent[max(ra, rb)] = min(ra, rb)
        return {k: find(k) for k in list(parent)}

    def relabel(self, labels, n, mp):
        if not mp:
            return
        L = labels[:n].numpy().view(np.uint32)
        out = np.array([mp.get(int(v), int(v)) for v in L.tolist()], dtype=np.uint32)
        labels[:n] = torch.from_numpy(out.view(np.int32))

    def split(self, feats, k, mp):
        f = _feats(feats[:k])
        inv = np.array([int(l) in mp for l in f["label"].tolist()], dtype=bool) if k else np.zeros(0, bool)
        kept = f[~inv]
        part = f[inv].copy()
        if len(part):
            part["label"] = [mp[int(l)] for l in part["label"].tolist()]
        return _feats_tensor(kept), len(kept), _feats_tensor(part), len(part)

    def fold(self, kept, nk, partials, Q, lo, hi, capacity):
        kept_f = _feats(kept[:nk]) if nk else np.zeros(0, FEAT)
        part = _feats(partials[:Q]) if Q else np.zeros(0, FEAT)
        part = part[(part["label"] >= lo) & (part["label"] < hi)]
        merged = {}
        for r in part:
            lab = int(r["label"])
            if lab not in merged:
                merged[lab] = r.copy()
            else:
                m = merged[lab]
                m["size"] += r["size"]
                m["toa_min"] = min(m["toa_min"], r["toa_min"])
                m["toa_max"] = max(m["toa_max"], r["toa_max"])
                for k in ("tot_sum", "sum_x", "sum_y", "sum_tot_x", "sum_tot_y"):
                    m[k] += r[k]
        allr = np.concatenate([kept_f, np.array(list(merged.values()), dtype=FEAT)]) if merged else kept_f
        allr = allr[np.argsort(allr["label"], kind="stable")]
        return _feats_tensor(allr), len(allr)


# ---- the protocol model
@dataclass
class ShardResult:
    labels: object        # this rank's labels (global input indices), n_r
    features: object      # records whose label falls in this rank's block, ascending
    n_clusters: int
    offset: int
    stats: dict


def model_cluster_sharded(hits, dt_max: int, comm, ops) -> ShardResult:
    """Run the sharded protocol for this rank's block ``hits`` ([n_r, 16] bytes)."""
    G, r = comm.world, comm.rank
    n = int(hits.shape[0]) if hits.dim() > 1 else int(hits.numel() // HIT_BYTES)
    hits = hits.reshape(n, HIT_BYTES) if n else hits
    sizes = [int(t[0].item()) for t in comm.allgather(ops.scalar_tensor([n]))]
    if min(sizes) == 0:
        raise ModelShardError("every rank needs at least one hit")
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    if offs[-1] >= 2**31:
        raise ModelShardError("sharded path supports < 2^31 hits in total")
    o_r = int(offs[r])
    mm = [tuple(int(v) for v in t.tolist()) for t in comm.allgather(ops.toa_range(hits, n))]
    for s in range(G):
        for t in range(s + 2, G):
            if mm[t][0] <= mm[s][1] + dt_max:
                raise ModelShardError(f"an edge could skip a rank ({s} -> {t}): blocks too small for dt_max")
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
