"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        k = d["Kernel Name"].split("(")[0]
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}.get(d["Metric Unit"], 1e-6)
        agg[k][0] += 1
        agg[k][1] += v * scale
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':45s} {'launches':>8s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:45s} {v[0]:8d} {v[1]:10.3f} {100*v[1]/tot:6.1f}%")
print(f"{'TOTAL':45s} {sum(v[0] for v in agg.values()):8d} {tot:10.3f}")
