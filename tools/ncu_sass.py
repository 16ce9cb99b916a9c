"""SASS instructions of an ncu report in address order with executed counts
(warp-level) and average active threads; optional address range filter.
   ncu_sass.py <rep> [min_count] [addr_lo addr_hi]"""
import csv, subprocess, sys
rep = sys.argv[1]
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
lo = int(sys.argv[3], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[4], 16) if len(sys.argv) > 4 else 1 << 62
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ix = {k: i for i, k in enumerate(hh)}
def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0
for r in rows[2:]:
    a = int(r[ix["Address"]], 16) & 0xfffff
    if not (lo <= a < hi):
        continue
    c = f(r, "Instructions Executed")
    if c >= mn:
        print(f"{a:05x} {c/1e6:8.2f}M thr {f(r,'Avg. Threads Executed'):5.1f} samp {f(r,'Warp Stall Sampling (All Samples)'):6.0f}  {r[ix['Source']][:100]}")
