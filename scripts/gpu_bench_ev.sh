#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for bd in ${BDS:-256 128}; do
  timeout 600 python bench.py --steps 2 --warmup 1 --particles 1e7 --no-cpu-baseline --no-e2e --no-ratio --block-dim=$bd > gpurun_out/bench_ev_$bd.log 2>&1
done
