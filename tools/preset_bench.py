"""Device-timed throughput of tpx_cluster_run on every BASELINE config at full
size (configs[4] as its per-GPU shard), with stage times.
    python tools/preset_bench.py [preset ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2412_11809_b200 as tpx
import tpxgen

SIZES = {"tiny": None, "lowflux": None, "mixed": None, "heavyion": None, "timepix4": 250_000_000}
MODE = os.environ.get("TPX_TILE_MODE", "auto")  # force a tile configuration (A/B)
presets = sys.argv[1:] or list(SIZES)
for preset in presets:
    p = tpxgen.PRESETS[preset]
    W, H = (448, 512) if preset == "timepix4" else (256, 256)
    h = tpxgen.generate(preset, n_hits=SIZES[preset])
    n = len(h)
    d = torch.from_numpy(h.view(np.uint8)).cuda()
    del h
    c = tpx.Clusterer(p["dt_max"], W, H)
    c.set_tile_mode(MODE)
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    feats = torch.empty((n, 64), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        c.run(d, labels=labels, features=feats)
    steps = 10
    s = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        _, _, k = c.run(d, labels=labels, features=feats)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    c.set_profiling(1)
    c.run(d, labels=labels, features=feats)
    st = c.stats()
    print(json.dumps({"preset": preset, "n_hits": n, "dt_max": p["dt_max"], "n_clusters": int(k),
                      "ms_per_run": round(ms, 3), "Mhit_s": round(n / ms / 1e3, 1),
                      "stage_ms": {kk: round(v, 3) for kk, v in st["stage_ms"].items()},
                      "tile_dense": st["tile_dense"], "sort_path": st["sort_path"],
                      "open_hits_frac": round(st["open_hits"] / n, 4), "tile_mode": MODE}), flush=True)
    c.close()
    del d, labels, feats
    torch.cuda.empty_cache()
