"""run_grouped on a preset (for ncu launch lists of the grouping kernels)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import tpxgen
import paper_2412_11809_b200 as tpx
preset = sys.argv[1] if len(sys.argv) > 1 else "mixed"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 50_000_000
h = tpxgen.generate(preset, n_hits=n)
d = torch.from_numpy(h.view(np.uint8)).cuda()
c = tpx.Clusterer(tpxgen.PRESETS[preset]["dt_max"])
for _ in range(2):
    c.run_grouped(d, n=n)
torch.cuda.synchronize()
print("ok")
