#!/bin/bash
# Round-2 first GPU call: parity tests, default bench line, compute-sanitizer on C1/C2.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_r02.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 900 > gpurun_out/pytest_gpu_base.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu_base.log
timeout 600 python bench.py > gpurun_out/bench_base.json 2> gpurun_out/bench_base.err
echo "bench exit $?" >> gpurun_out/bench_base.err
for tool in memcheck synccheck racecheck; do
  for cfg in c1 c2; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize.py --cfg $cfg --n 200000 \
      > gpurun_out/sanitize_${tool}_${cfg}.log 2>&1
    echo "exit $?" >> gpurun_out/sanitize_${tool}_${cfg}.log
  done
done
echo done
