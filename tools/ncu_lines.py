"""Per-source-line totals (instructions executed, stall samples) from an ncu report."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = None
res = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if hdr and r and r[0] not in ("", "Function Name") and len(r) > 8:
        try:
            inst = float(r[7]); samp = float(r[4]); thr = float(r[10])
        except ValueError:
            continue
        res.append((fname, r[0], inst, samp, thr, r[1].strip()[:80]))
ti = sum(x[2] for x in res); ts = sum(x[3] for x in res)
print(f"total inst {ti:.3e} samples {ts:.0f}")
for key, name in ((2, "inst"), (3, "samples")):
    print("--- by", name)
    for x in sorted(res, key=lambda x: -x[key])[:top]:
        print(f"{x[0]}:{x[1]:>4} inst {x[2]:11.0f} ({100*x[2]/ti:4.1f}%) samp {x[3]:7.0f} ({100*x[3]/ts:4.1f}%) thr {x[4]:5.1f} | {x[5]}")
