"""CPU reference implementation of the sharded protocol's compute steps.

TEST INFRASTRUCTURE: it lets the distributed protocol in
paper_2412_11809_b200/sharded.py (halo selection, exchanges, pair union,
relabel, partial folding) run on CPU tensors with a gloo process group or
in-process threads, with every per-rank compute step done here with numpy and
the oracle instead of the CUDA kernels.  The protocol code itself is the
product's; only the ``ops`` backend is swapped.
"""
from __future__ import annotations

import numpy as np
import torch

import oracle
from tests import pins
from tpxgen import HIT_DTYPE

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
