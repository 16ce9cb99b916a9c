#!/bin/bash
# A/B of prebuilt libraries (abl/A.so = baseline, abl/B.so = candidate, or
# LIBS="A B C ..." for abl/<name>.so): fast GPU parity tests on the last one,
# then the kernel-only bench alternating over the libraries twice, and the
# preset bench on each.   tools/ab_lib.sh [pytest -k expr] [presets]
mkdir -p gpurun_out
LIB=paper_2412_11809_b200/lib/libtpxcluster.so
K=${1:-"not slow"}
LIBS=${LIBS:-"A B"}
LAST=${LIBS##* }
cp abl/$LAST.so $LIB
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q -k "$K" > gpurun_out/ab_pt.log 2>&1; echo "pytest($LAST)=$?"; tail -2 gpurun_out/ab_pt.log
for r in 1 2; do for v in $LIBS; do
cp abl/$v.so $LIB
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ab_$v$r.json 2> gpurun_out/ab_$v$r.err
python -c "import json;d=json.load(open('gpurun_out/ab_$v$r.json'));print('$v$r',d['value'],d['ms_per_step'],d['stage_ms'],d['parity']['status'])" || tail -3 gpurun_out/ab_$v$r.err
done; done
for v in $LIBS; do
cp abl/$v.so $LIB
timeout 900 python tools/preset_bench.py ${2:-timepix4 heavyion lowflux} 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print('$v',d['preset'],d['ms_per_run'],d['Mhit_s'],d['stage_ms'])
    except Exception: pass"
done
cp abl/$LAST.so $LIB
