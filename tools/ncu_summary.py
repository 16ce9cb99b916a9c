"""Summarise an ncu report: key raw metrics + top SASS lines by instructions/stalls."""
import csv, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct"]
for r in rows[2:]:
    d = dict(zip(h, r))
    print({k: d.get(k) for k in keys})
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(d[k]) for k in h
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and d[k] not in ("", "n/a")}
    tot = sum(st.values()) or 1
    print("stalls:", ", ".join(f"{k} {100*v/tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
hh = rows[1]
ix = {k: i for i, k in enumerate(hh)}
data = rows[2:]
def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0
ti = sum(f(r, "Instructions Executed") for r in data)
ts = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"total warp-inst {ti:.3e}  samples {ts:.0f}")
for key in ("Warp Stall Sampling (All Samples)", "Instructions Executed"):
    print("--- top by", key)
    for r in sorted(data, key=lambda r: -f(r, key))[:top]:
        print(f"{r[ix['Address']][-5:]} inst {f(r,'Instructions Executed'):11.0f} thr {f(r,'Avg. Threads Executed'):5.1f} "
              f"samp {f(r,'Warp Stall Sampling (All Samples)'):7.0f}  {r[ix['Source']][:90]}")
