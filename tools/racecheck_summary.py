"""Run tests/native/abi_run under compute-sanitizer racecheck on a few cases
and aggregate the reported shared-memory hazards by source line pair.

    python tools/racecheck_summary.py [out.txt]
"""
import collections
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import tpxgen  # noqa: E402
import test_gpu_sanitizer as T  # noqa: E402


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else None
    from paper_2412_11809_b200 import build

    lib = build.build()
    d = tempfile.mkdtemp()
    exe = os.path.join(d, "abi_run")
    cuda = "/usr/local/cuda"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-I", os.path.join(ROOT, "include"), "-I", f"{cuda}/include",
                           os.path.join(ROOT, "tests", "native", "abi_run.c"), "-L", os.path.dirname(lib),
                           "-ltpxcluster", "-L", f"{cuda}/lib64", "-lcudart", f"-Wl,-rpath,{os.path.dirname(lib)}",
                           "-o", exe])
    lines = []
    for case, (make, dt, W, H, mode, variant) in T.CASES.items():
        h = make()
        hp = os.path.join(d, "h.bin")
        h.tofile(hp)
        r = subprocess.run([T.SANITIZER, "--tool", "racecheck", "--racecheck-report", "all", "--print-limit", "100000",
                            exe, hp, str(dt), str(W), str(H), os.path.join(d, "l"), os.path.join(d, "f"), str(mode),
                            str(variant)], capture_output=True, text=True, timeout=1800)
        txt = r.stdout + r.stderr
        agg = collections.Counter()
        cur = None
        for ln in txt.splitlines():
            m = re.search(r"(Warning|Error).*Potential (\w+) hazard", ln)
            if m:
                cur = [m.group(1), m.group(2)]
                continue
            m = re.search(r"(Write|Read) Thread .* at (.*?)\+0x[0-9a-f]+ in (\S+:\d+)", ln)
            if m and cur is not None:
                cur.append(f"{m.group(1)} {m.group(3)} ({m.group(2)[:40]})")
                if len(cur) == 4:
                    agg[tuple(cur)] += 1
                    cur = None
        summ = [l for l in txt.splitlines() if "SUMMARY" in l]
        lines.append(f"== {case}: {summ}")
        for k, v in agg.most_common(30):
            lines.append(f"  {v:7d}  {' | '.join(k)}")
    s = "\n".join(lines)
    print(s)
    if out:
        open(out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
