"""Per-kernel DRAM bytes and time for every launch in an ncu CSV captured with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum;
prints per-kernel totals and the whole-step DRAM GB/s."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = None
rec = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < len(hdr):
        continue
    k = r[hdr["Kernel Name"]].split("(")[0]
    name, unit = r[hdr["Metric Name"]], r[hdr["Metric Unit"]]
    v = float(r[hdr["Metric Value"]].replace(",", ""))
    scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0,
             "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1.0)
    rec[k][name] += v * scale
    if name == "gpu__time_duration.sum":
        cnt[k] += 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
tot_ms = sum(d["gpu__time_duration.sum"] for d in rec.values()) / steps
tot_b = sum(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"] for d in rec.values()) / steps
print(f"{'kernel':45s} {'ms/step':>9s} {'GB/step':>8s} {'GB/s':>8s}")
for k, d in sorted(rec.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    ms = d["gpu__time_duration.sum"] / steps
    gb = (d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]) / steps / 1e9
    print(f"{k[:45]:45s} {ms:9.3f} {gb:8.3f} {gb / (ms * 1e-3) if ms else 0:8.1f}")
print(f"{'WHOLE STEP (serialised launches)':45s} {tot_ms:9.3f} {tot_b/1e9:8.3f} {tot_b/1e9/(tot_ms*1e-3):8.1f}")
