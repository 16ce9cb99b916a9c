"""Regenerate profiles/traffic.json (bench.py's roofline.traffic / issue
inputs) from an ncu --set full report of the bench workload:
dram__bytes_read.sum + dram__bytes_write.sum and smsp__inst_executed.sum per
launch of the tile kernel ("tile_cc" stage) and the window sort ("sort").
    python tools/traffic_from_ncu.py report.ncu-rep "<source note>" """
import csv
import json
import os
import subprocess
import sys

rep, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
out = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"]
    stage = "tile_cc" if ("k_tile_csr" in name or "k_tile_cell" in name or "k_tile_cc" in name) else "sort" if "k_window_sort" in name else None
    if not stage or stage in out:
        continue
    out[stage] = int(float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"]))
    out[stage + "_warp_inst"] = int(float(d["smsp__inst_executed.sum"]))
    out[stage + "_kernel"] = name.split("(")[0]
out["_source"] = (f"ncu --set full {os.path.basename(rep)} {note}: dram__bytes_read.sum + dram__bytes_write.sum "
                  "per launch; *_warp_inst = smsp__inst_executed.sum per launch")
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
with open(os.path.join(root, "profiles", "traffic.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
