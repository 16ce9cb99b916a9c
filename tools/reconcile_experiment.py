"""Δt-relaxation reconciliation experiment:
on Pb data the paper's local-neighbourhood clustering (variant (iii)(a))
disagreed with Tracklab (global neighbourhood, (iii)(b)) at Δt_max = 200 ns
and matched it exactly at 600 ns.  Synthetic analogue: heavy-ion blob streams
(and a blob + track mix), clustered on the GPU by (b) at 200 ns (128 ticks)
and by (a) at 200, 400 and 600 ns (128 / 256 / 384 ticks).  Reported per
pair: the hit-weighted mean IoU of every (b)-cluster with its best-matching
(a)-cluster, and the fraction of (b)-clusters reproduced exactly.  A sample
of each GPU partition is checked against the oracle first.

    python tools/reconcile_experiment.py [n_hits]   (one JSON line per workload)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2412_11809_b200 as tpx
import tpxgen

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
WORKLOADS = {
    "heavyion": dict(preset="heavyion"),
    "pb_mix": dict(preset="heavyion", frac_blob=0.5, frac_track=0.3, frac_dot=0.2, seed=41),
}


def gpu_labels(h, dt, variant):
    c = tpx.Clusterer(dt, variant=variant)
    d = torch.from_numpy(h.view(np.uint8)).cuda()
    labels, _, _ = c.run(d)
    torch.cuda.synchronize()
    return labels.cpu().numpy().view(np.uint32).astype(np.int64)


def compare(lb, la):
    """IoU of each (b)-cluster with its best (a)-cluster, hit-weighted; exact matches."""
    n_ = len(lb)
    size_b = np.bincount(lb, minlength=n_)
    size_a = np.bincount(la, minlength=n_)
    pair = lb * n_ + la
    up, cnt = np.unique(pair, return_counts=True)
    pb, pa = up // n_, up % n_
    order = np.lexsort((-cnt, pb))  # per b-cluster, largest intersection first
    pb, pa, cnt = pb[order], pa[order], cnt[order]
    first = np.concatenate([[True], pb[1:] != pb[:-1]])
    pb, pa, inter = pb[first], pa[first], cnt[first]
    union = size_b[pb] + size_a[pa] - inter
    iou = inter / union
    w = size_b[pb]
    exact = (inter == size_b[pb]) & (inter == size_a[pa])
    return {"iou_hit_weighted": round(float((iou * w).sum() / w.sum()), 6),
            "clusters_b": int(len(pb)), "exact_fraction": round(float(exact.mean()), 6),
            "hits_in_exact_clusters": round(float(w[exact].sum() / w.sum()), 6)}


for name, wl in WORKLOADS.items():
    preset = wl.pop("preset")
    h = tpxgen.generate(preset, n_hits=n, **wl)
    # parity spot check on a 200k-hit prefix (the GPU paths are pinned by the tests)
    hp = h[:200_000]
    assert np.array_equal(gpu_labels(hp, 128, tpx.VARIANT_LOCAL), oracle.cluster(hp, 128)[0])
    assert np.array_equal(gpu_labels(hp, 128, tpx.VARIANT_GLOBAL), oracle.cluster_streaming(hp, 128, 1))
    lb = gpu_labels(h, 128, tpx.VARIANT_GLOBAL)
    out = {"workload": name, "n_hits": n, "reference": "(iii)(b) global, dt = 200 ns (128 ticks)"}
    for dt_ns, dt in ((200, 128), (400, 256), (600, 384)):
        out[f"local_{dt_ns}ns"] = compare(lb, gpu_labels(h, dt, tpx.VARIANT_LOCAL))
    print(json.dumps(out))
