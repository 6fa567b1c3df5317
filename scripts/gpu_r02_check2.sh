#!/bin/bash
# Ring-protocol fix check: stress, per-file GPU tests with their own timeouts, bench, racecheck on the ring.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 900 python scripts/stress_ring.py 20 > gpurun_out/stress_ring.log 2>&1; echo "exit $?" >> gpurun_out/stress_ring.log
for f in test_gpu_parity test_gpu_flags test_distributed_gpu test_gpu_parity_large; do
  timeout 1500 python -m pytest tests/$f.py -v -x --timeout 600 --durations=15 > gpurun_out/pytest_$f.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_$f.log
done
timeout 900 python bench.py > gpurun_out/bench_fix.json 2> gpurun_out/bench_fix.err; echo "bench exit $?" >> gpurun_out/bench_fix.err
for s in block rounds rect-ring; do
  timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python scripts/sanitize.py --cfg c1 --n 200000 --scheds $s \
    > gpurun_out/racecheck2_c1_$s.log 2>&1
  echo "exit $?" >> gpurun_out/racecheck2_c1_$s.log
done
echo done
