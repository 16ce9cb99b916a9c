#!/bin/bash
# parity subset + mixed bench + preset bench: tools/ab_presets.sh [pytest -k expr] [presets]
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "${1:-not slow}" > gpurun_out/ab_pt.log 2>&1; echo "pytest=$?"; tail -2 gpurun_out/ab_pt.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ab_b1.json 2> gpurun_out/ab_b1.err
python -c "import json;d=json.load(open('gpurun_out/ab_b1.json'));print(d['value'],d['ms_per_step'],d['stage_ms'],d.get('parity',{}).get('status'))" || tail -5 gpurun_out/ab_b1.err
timeout 900 python tools/preset_bench.py ${2:-timepix4 heavyion lowflux} 2>&1 | tail -3
