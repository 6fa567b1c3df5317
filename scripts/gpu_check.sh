#!/bin/bash
# First GPU round: smoke, GPU parity tests, a short bench.  Outputs under gpurun_out/.
set -x
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 2 --warmup 1 --particles 1e7 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1
echo "bench exit $?" >> gpurun_out/bench_small.log
