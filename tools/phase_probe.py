"""Run the path with profiling on and print stage times + k_tile_cc phase shares."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import tpxgen
import paper_2412_11809_b200 as tpx

preset = sys.argv[1] if len(sys.argv) > 1 else "mixed"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20_000_000
p = tpxgen.PRESETS[preset]
W, H = (448, 512) if preset == "timepix4" else (256, 256)
h = tpxgen.generate(preset, n_hits=n)
d = torch.from_numpy(h.view(np.uint8)).cuda()
c = tpx.Clusterer(p["dt_max"], W, H)
for _ in range(2):
    c.run(d)
c.set_profiling(2)
c.run(d)
st = c.stats()
names = ["meta", "stage+index", "scatter+rank", "search+union", "flatten", "sizes+pairs", "compact", "features", "outputs"]
cyc = st["tile_phase_cycles"][:9]
tot = sum(cyc) or 1
print(preset, n, {k: round(v, 3) for k, v in st["stage_ms"].items()})
print("open_hits %.3f%%  overflow %.3f%%  pairs %d  sort_path %d" % (100 * st["open_hits"] / n, 100 * st["overflow_hits"] / n, st["cross_pairs"], st["sort_path"]))
print("tile phases:", ", ".join(f"{nm} {100*v/tot:.1f}%" for nm, v in zip(names, cyc)))
