#!/bin/bash
# A/B of an environment switch: tools/ab_env.sh VAR [pytest -k expr]
V=$1; K=${2:-"presets or forced or sizes"}
mkdir -p gpurun_out
env $V=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/ab_pt.log 2>&1; echo "pytest($V)=$?"; tail -1 gpurun_out/ab_pt.log
for on in 0 1; do
if [ $on = 1 ]; then export $V=1; fi
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ab_e$on.json 2> gpurun_out/ab_e$on.err
python -c "import json;d=json.load(open('gpurun_out/ab_e$on.json'));print('$V=$on',d['value'],d['ms_per_step'],d['stage_ms'])" || tail -3 gpurun_out/ab_e$on.err
done
