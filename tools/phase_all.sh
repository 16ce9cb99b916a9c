#!/bin/bash
# Stage times + k_tile_cc phase shares on every preset (profiling level 2).
mkdir -p gpurun_out
for p in "mixed 50000000" "timepix4 50000000" "heavyion 20000000" "lowflux 10000000"; do
  timeout 300 python tools/phase_probe.py $p >> gpurun_out/phases.log 2>&1
done
