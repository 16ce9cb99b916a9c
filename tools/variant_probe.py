"""One variant run (global / static) on a preset, for ncu launch lists."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import tpxgen
import paper_2412_11809_b200 as tpx
variant = sys.argv[1] if len(sys.argv) > 1 else "static"
preset = sys.argv[2] if len(sys.argv) > 2 else "mixed"
n = int(sys.argv[3]) if len(sys.argv) > 3 else 20_000_000
h = tpxgen.generate(preset, n_hits=n)
d = torch.from_numpy(h.view(np.uint8)).cuda()
c = tpx.Clusterer(tpxgen.PRESETS[preset]["dt_max"], variant={"global": tpx.VARIANT_GLOBAL, "static": tpx.VARIANT_STATIC}[variant])
for _ in range(2):
    c.run(d)
torch.cuda.synchronize()
print("ok", c.stats()["sort_retries"])
