#!/bin/bash
# Lap-tagged ring check: stress (incl. DP + mesh), GPU tests per file (thread-method timeouts), bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 600 python scripts/stress_ring.py 10 > gpurun_out/stress_ring3.log 2>&1; echo "exit $?" >> gpurun_out/stress_ring3.log
for f in test_gpu_parity test_gpu_flags test_gpu_parity_large test_distributed_gpu; do
  timeout 1200 python -m pytest tests/$f.py -v -x --timeout 300 --timeout_method thread --durations=10 > gpurun_out/pytest3_$f.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest3_$f.log
done
timeout 900 python bench.py > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "bench exit $?" >> gpurun_out/bench3.err
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python scripts/sanitize.py --cfg c1 --n 200000 --scheds block \
    > gpurun_out/racecheck3_c1_block.log 2>&1; echo "exit $?" >> gpurun_out/racecheck3_c1_block.log
echo done
