#!/bin/bash
# ncu launch list (per-kernel durations) of one preset run: tools/preset_launches.sh <preset> [tag]
P=${1:-heavyion}; T=${2:-x}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${P}_${T}.csv \
  python tools/preset_bench.py $P > gpurun_out/pl_${P}.log 2>&1; echo ncu=$?
python tools/summarize_launches.py gpurun_out/launches_${P}_${T}.csv | head -30
