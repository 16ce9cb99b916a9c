#!/bin/bash
# Window-sort A/B: parity subset, mixed bench with TPX_WSORT_ALT=0/1, preset bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${1:-not slow}" > gpurun_out/ab_pt.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/ab_pt.log
for alt in 0 1; do
TPX_WSORT_ALT=$alt timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ab_s$alt.json 2> gpurun_out/ab_s$alt.err
python -c "import json;d=json.load(open('gpurun_out/ab_s$alt.json'));print('alt=$alt',d['value'],d['ms_per_step'],d['stage_ms'])" || tail -3 gpurun_out/ab_s$alt.err
done
timeout 900 python tools/preset_bench.py ${2:-timepix4 heavyion lowflux} 2>&1 | tail -4
