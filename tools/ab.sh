#!/bin/bash
# A/B on the GPU box: parity subset + kernel-only bench (stage times) + optional ncu of the tile kernel.
#   tools/ab.sh [pytest -k expr] [ncu]
mkdir -p gpurun_out
K=${1:-"not slow"}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "$K" > gpurun_out/ab_pt.log 2>&1; echo "pytest=$?"; tail -5 gpurun_out/ab_pt.log
for i in 1 2; do
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ab_b$i.json 2> gpurun_out/ab_b$i.err; echo "bench=$?"
python -c "import json;d=json.load(open('gpurun_out/ab_b$i.json'));print(d['value'],d['ms_per_step'],d['stage_ms'],d.get('parity',{}).get('status'))" || tail -5 gpurun_out/ab_b$i.err
done
if [ -n "$2" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_tile_c" -s 3 -c 1 \
  -o gpurun_out/ab_full python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ab_ncu.log 2>&1; echo "ncu=$?"
fi
