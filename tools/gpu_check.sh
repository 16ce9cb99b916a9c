#!/bin/bash
# One GPU round trip: smoke, GPU parity tests, short bench (+ optional ncu of a kernel).
#   tools/gpu_check.sh [fast|full] [ncu-kernel-regex]
mkdir -p gpurun_out
MODE=${1:-fast}
SEL="gpu and not slow"; [ "$MODE" = full ] && SEL="gpu"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1500 python -m pytest tests -m "$SEL" -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench=$?"
if [ -n "$2" ]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k "regex:$2" -s 1 -c 1 -o gpurun_out/prof \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --n-hits 20000000 > gpurun_out/ncu.log 2>&1; echo "ncu=$?"
fi
