"""Repro: wide-ToA input in each tile mode (run under compute-sanitizer)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import tpxgen
import paper_2412_11809_b200 as tpx
mode = sys.argv[1] if len(sys.argv) > 1 else "auto"
h = tpxgen.generate("mixed", n_hits=50_000)
h["toa"][::7] += np.uint64(1 << 40)
h["toa"] += np.uint64((1 << 47))
c = tpx.Clusterer(320)
c.set_tile_mode(mode)
d = torch.from_numpy(h.view(np.uint8)).cuda()
try:
    labels, feats, k = c.run(d)
    torch.cuda.synchronize()
    print(mode, "ok k=", k, c.stats())
except Exception as e:
    print(mode, "FAIL", e, c.stats())
