#!/bin/bash
# parity tests (short) + the four schedulers/trackers on C3 (1e7 histories)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests -m gpu -x -q --timeout 600 -k "not full_size" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
for v in "warp:--scheduler warp" "block:--scheduler block" "history:--scheduler history" "rect:--tracker rect"; do
  name=${v%%:*}; args=${v#*:}
  timeout 600 python bench.py --steps 2 --warmup 1 --particles 1e7 --no-cpu-baseline --no-e2e $args ${BENCH_ARGS} > gpurun_out/bench_$name.log 2>&1
done
