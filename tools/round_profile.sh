#!/bin/bash
# Round evidence: GPU tests, bench, launch list and a full ncu capture of the
# two dominant kernels at the bench size.   tools/round_profile.sh <tag>
TAG=${1:-r01}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke=$?"
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; echo "bench=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ncu_launch.log 2>&1; echo "ncu_launch=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:k_tile_csr|k_tile_cell|k_window_sort" -s 6 -c 2 \
  -o gpurun_out/full_${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-grouped --no-variants > gpurun_out/ncu_full.log 2>&1; echo "ncu_full=$?"
