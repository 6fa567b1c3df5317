#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -x --timeout 600 -k "async" > gpurun_out/pytest_async.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_async.log
for s in async block warp; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --scheduler $s > gpurun_out/bench_s_$s.json 2>&1
done
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --scheduler warp --config c4 > gpurun_out/bench_s_warp_c4.json 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --scheduler async --config c4 > gpurun_out/bench_s_async_c4.json 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --scheduler block --config c4 > gpurun_out/bench_s_block_c4.json 2>&1
echo done
