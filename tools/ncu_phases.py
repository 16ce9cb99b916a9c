"""Per-phase instruction / stall totals of a tile kernel from an ncu report:
SASS lines are attributed to the nearest preceding line of the kernel source
file (inlined helpers inherit the caller's line), then bucketed by the
TPX_PHASE markers' line numbers.   ncu_phases.py <rep> <file.cuh>"""
import csv, re, subprocess, sys
rep, src = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
# source view: file blocks, each with lines (Line No, Source, ...) -- we need SASS->line mapping;
# use the sass+cuda print: rows with 'Address' columns carry the source line in 'Source' for cuda rows.
lines = open(src).read().splitlines()
marks = [(i + 1, m.group(1)) for i, l in enumerate(lines) for m in [re.search(r"TPX_PHASE\((\d+)\)", l)] if m]
def phase_of(ln):
    p = "0"
    for mln, k in marks:
        if ln > mln:
            p = str(int(k) + 1) if False else k
    # the phase ending at the first marker after ln
    for mln, k in marks:
        if ln <= mln:
            return k
    return "end"
fname = None; hdr = None; per = {}
cur_line = 0
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]; hdr = None; continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}; continue
    if hdr is None or not r or fname != src.split("/")[-1]:
        continue
    try:
        ln = int(r[0]); inst = float(r[hdr["Instructions Executed"]]); samp = float(r[hdr["Warp Stall Sampling (All Samples)"]])
    except (ValueError, KeyError):
        continue
    k = phase_of(ln)
    a = per.setdefault(k, [0.0, 0.0]); a[0] += inst; a[1] += samp
ti = sum(v[0] for v in per.values()) or 1; ts = sum(v[1] for v in per.values()) or 1
for k, v in sorted(per.items(), key=lambda x: x[0]):
    print(f"phase<= {k:>4}: inst {v[0]:12.0f} ({100*v[0]/ti:5.1f}%)  samples {v[1]:8.0f} ({100*v[1]/ts:5.1f}%)")
