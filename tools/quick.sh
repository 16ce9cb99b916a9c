#!/bin/bash
# Quick A/B on the GPU box: parity subset + kernel-only bench (stage times).
#   tools/quick.sh [pytest -k expr]
mkdir -p gpurun_out
K=${1:-"not slow"}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/q_pt.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/q_pt.log
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/q_b$i.json 2> gpurun_out/q_b$i.err; echo "bench=$?"
python -c "import json;d=json.load(open('gpurun_out/q_b$i.json'));print(d['value'],d['ms_per_step'],d['stage_ms'])"
done
