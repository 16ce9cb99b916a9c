#!/bin/bash
# Iteration loop for the tile kernel: targeted parity tests, phase probe, one ncu capture.
#   tools/cell_iter.sh <tag> [kernel-regex]
TAG=${1:-it}; K=${2:-k_tile_cell}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "forced or presets or sizes or fuzz or examples" > gpurun_out/pt_$TAG.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pt_$TAG.log
rm -f gpurun_out/phases.log; tools/phase_all.sh; cp gpurun_out/phases.log gpurun_out/phases_$TAG.log; cat gpurun_out/phases.log
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$K" -s 3 -c 1 -o gpurun_out/$TAG python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants --no-stream --n-hits 20000000 > gpurun_out/ncu_$TAG.log 2>&1; echo ncu=$?
