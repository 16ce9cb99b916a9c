"""Independent checks used to pin the oracle (and, at full size, the GPU path).

Nothing here calls the oracle or the CUDA path: every function is a separate
restatement of what the paper fixes, using numpy / scipy library routines:

* ``brute_edges``      O(n^2) pairwise enumeration of the edge predicate
                       (§2 (ii) l.35 + (iii)(a) l.39, §4.1 l.217).
* ``indexed_edges``    the same edge set by sorting + searchsorted (O(n log n)),
                       for certificate checks on larger inputs.
* ``cc_labels``        connected components via scipy.sparse.csgraph,
                       canonicalised to the smallest member index (reading R6).
* ``features_from_labels``  numpy bincount / minimum.at / maximum.at.
* ``paper_sequential`` the paper's own sequential method: hits in ToA order,
                       last hit per pixel, find on the 9 neighbour pixels, union
                       (§4.1 Step 4 l.171, l.215-221), pure Python.
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import connected_components

FEAT_FIELDS = ("label", "size", "toa_min", "toa_max", "tot_sum", "sum_x", "sum_y",
               "sum_tot_x", "sum_tot_y")


def brute_edges(h, dt: int):
    """All pairs i < j with Chebyshev distance <= 1 and |dToA| <= dt."""
    n = len(h)
    x = h["x"].astype(np.int64)
    y = h["y"].astype(np.int64)
    t = h["toa"].astype(np.int64)
    I, J = [], []
    step = max(1, 4_000_000 // max(n, 1))
    for a in range(0, n, step):
        b = min(n, a + step)
        ok = (np.abs(x[a:b, None] - x[None, :]) <= 1) & (np.abs(y[a:b, None] - y[None, :]) <= 1) \
            & (np.abs(t[a:b, None] - t[None, :]) <= dt)
        ii, jj = np.nonzero(ok)
        ii = ii + a
        keep = ii < jj
        I.append(ii[keep])
        J.append(jj[keep])
    if not I:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(I), np.concatenate(J)


def indexed_edges(h, dt: int, width: int):
    """Same edge set as brute_edges, found per pixel offset with searchsorted."""
    n = len(h)
    x = h["x"].astype(np.int64)
    y = h["y"].astype(np.int64)
    t = h["toa"].astype(np.int64)
    pix = y * (width + 2) + x           # padded row stride: no wraparound aliasing
    key_order = np.lexsort((np.arange(n), t, pix))
    SH = np.int64(1) << 40
    assert n == 0 or int(t.max()) + dt < int(SH), "toa too large for the combined key"
    skey = pix[key_order] * SH + t[key_order]
    I, J = [], []
    for dy in (-1, 0, 1):
        for dx in (-1, 0, 1):
            qpix = (y + dy) * (width + 2) + (x + dx)
            valid = (x + dx >= 0) & (x + dx < width) & (y + dy >= 0)
            # window [t - dt, t + dt] inside bucket qpix, located in the
            # (pix, toa)-sorted order via a combined search
            lo = np.searchsorted(skey, qpix * SH + np.maximum(t - dt, 0), "left")
            hi = np.searchsorted(skey, qpix * SH + (t + dt), "right")
            cnt = np.where(valid, hi - lo, 0)
            src = np.repeat(np.arange(n), cnt)
            starts = np.repeat(lo, cnt)
            offs = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            dst = key_order[starts + offs]
            keep = src < dst
            I.append(src[keep])
            J.append(dst[keep])
    return np.concatenate(I), np.concatenate(J)


def cc_labels(n: int, I, J) -> np.ndarray:
    """Connected components (scipy), label = smallest member index."""
    if n == 0:
        return np.zeros(0, np.uint32)
    g = sp.coo_matrix((np.ones(len(I), np.int8), (I, J)), shape=(n, n)).tocsr()
    _, comp = connected_components(g, directed=False)
    first = np.full(comp.max() + 1, n, dtype=np.int64)
    np.minimum.at(first, comp, np.arange(n))
    return first[comp].astype(np.uint32)


def features_from_labels(h, labels) -> dict:
    """Per-cluster features, ascending label (numpy reductions)."""
    labels = np.asarray(labels, np.int64)
    uniq = np.unique(labels)
    k = np.searchsorted(uniq, labels)
    m = len(uniq)
    tot = h["tot"].astype(np.uint64)
    x = h["x"].astype(np.uint64)
    y = h["y"].astype(np.uint64)
    toa = h["toa"].astype(np.uint64)
    f = {
        "label": uniq.astype(np.uint32),
        "size": np.bincount(k, minlength=m).astype(np.uint32),
        "tot_sum": np.zeros(m, np.uint64), "sum_x": np.zeros(m, np.uint64),
        "sum_y": np.zeros(m, np.uint64), "sum_tot_x": np.zeros(m, np.uint64),
        "sum_tot_y": np.zeros(m, np.uint64),
        "toa_min": np.full(m, np.iinfo(np.uint64).max, np.uint64),
        "toa_max": np.zeros(m, np.uint64),
    }
    np.add.at(f["tot_sum"], k, tot)
    np.add.at(f["sum_x"], k, x)
    np.add.at(f["sum_y"], k, y)
    np.add.at(f["sum_tot_x"], k, tot * x)
    np.add.at(f["sum_tot_y"], k, tot * y)
    np.minimum.at(f["toa_min"], k, toa)
    np.maximum.at(f["toa_max"], k, toa)
    return f


def assert_features_equal(feats, ref: dict, ctx: str = ""):
    assert len(feats) == len(ref["label"]), f"{ctx}: cluster count {len(feats)} vs {len(ref['label'])}"
    for name in FEAT_FIELDS:
        a = np.asarray(feats[name]).astype(np.uint64)
        b = np.asarray(ref[name]).astype(np.uint64)
        bad = np.nonzero(a != b)[0]
        assert len(bad) == 0, f"{ctx}: field {name} differs at {bad[:5]} ({a[bad[:5]]} vs {b[bad[:5]]})"


def paper_sequential(h, dt: int, width: int, height: int) -> np.ndarray:
    """PAPER.md §4.1: hits in (toa, index) order; per pixel the last hit;
    findNeighborClusters = find() on the 9 neighbour pixels' last hits
    (l.217); union (l.215-221).  Exact for CC under reading R2."""
    n = len(h)
    order = np.lexsort((np.arange(n), h["toa"].astype(np.int64)))
    parent = list(range(n))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    last = {}
    xs, ys, ts = h["x"].tolist(), h["y"].tolist(), h["toa"].tolist()
    for i in order.tolist():
        xi, yi, ti = xs[i], ys[i], ts[i]
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                q = (xi + dx, yi + dy)
                j = last.get(q)
                if j is not None and ti - ts[j] <= dt:
                    a, b = find(i), find(j)
                    if a != b:
                        parent[max(a, b)] = min(a, b)
        last[(xi, yi)] = i
    roots = [find(i) for i in range(n)]
    first = {}
    for i, r in enumerate(roots):
        first.setdefault(r, i)
    return np.array([first[r] for r in roots], dtype=np.uint32)


def is_refinement(fine, coarse) -> bool:
    """Every class of `fine` lies inside one class of `coarse`."""
    fine = np.asarray(fine)
    coarse = np.asarray(coarse)
    m = {}
    for a, b in zip(fine.tolist(), coarse.tolist()):
        if m.setdefault(a, b) != b:
            return False
    return True


def streaming_last_writer(h, dt: int, variant: int) -> np.ndarray:
    """Variants (iii)(b) GLOBAL (variant 1) / (iii)(c) STATIC (variant 2) with
    SPEC's per-pixel reference matrix ("PixelRefMatrix"): hits in
    (toa, index) order; for each of the 9 pixels only the cluster of the
    pixel's LAST hit is a candidate; it is joinable if toa - maxToA (b) /
    toa - minToA (c) <= dt; the hit joins and merges every joinable
    candidate.  Structurally different from the oracle (reading R21: every
    cluster with any member on the 9 pixels).  The two readings coincide:
    a hit on pixel p that did not join cluster A (which has a member on p)
    found A non-joinable, and A can never become joinable again (maxToA /
    minToA only change when a hit joins), so an overwritten reference only
    ever hides a dead cluster."""
    n = len(h)
    order = np.lexsort((np.arange(n), h["toa"].astype(np.int64)))
    parent = list(range(n))
    cmin, cmax, cidx = {}, {}, {}

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    last = {}
    xs, ys, ts = h["x"].tolist(), h["y"].tolist(), h["toa"].tolist()
    for i in order.tolist():
        xi, yi, ti = xs[i], ys[i], ts[i]
        cands = set()
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                j = last.get((xi + dx, yi + dy))
                if j is None:
                    continue
                r = find(j)
                ref = cmax[r] if variant == 1 else cmin[r]
                if ti - ref <= dt:
                    cands.add(r)
        root = i
        cmin[i], cmax[i], cidx[i] = ti, ti, i
        for r in cands:
            a, b = min(root, r), max(root, r)
            parent[b] = a
            cmin[a], cmax[a], cidx[a] = min(cmin[a], cmin[b]), max(cmax[a], cmax[b]), min(cidx[a], cidx[b])
            root = a
        last[(xi, yi)] = i
    return np.array([cidx[find(i)] for i in range(n)], dtype=np.uint32)
