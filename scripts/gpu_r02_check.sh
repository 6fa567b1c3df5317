#!/bin/bash
# Round-2 check: new GPU tests (flags, large batches, 2-rank device path), racecheck per scheduler, bench.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_flags.py tests/test_distributed_gpu.py tests/test_gpu_parity_large.py tests/test_gpu_parity.py -q --timeout 1200 -x > gpurun_out/pytest_gpu_new.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_new.log
timeout 600 python bench.py > gpurun_out/bench_new.json 2> gpurun_out/bench_new.err
echo "bench exit $?" >> gpurun_out/bench_new.err
for s in block rounds warp history dp rect; do
  timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python scripts/sanitize.py --cfg c1 --n 200000 --scheds $s \
    > gpurun_out/racecheck_c1_$s.log 2>&1
  echo "exit $?" >> gpurun_out/racecheck_c1_$s.log
done
echo done
