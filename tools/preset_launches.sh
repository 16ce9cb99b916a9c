#!/bin/bash
# Per-kernel launch list (ncu gpu__time_duration) of one clustering run on a preset.
#   tools/preset_launches.sh <preset> <n_hits> <tag>
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$3.csv \
  python tools/phase_probe.py $1 $2 > gpurun_out/launches_$3.log 2>&1
python tools/summarize_launches.py gpurun_out/launches_$3.csv > gpurun_out/launches_$3.txt 2>&1
