#!/bin/bash
# Build check on the GPU: ring stress, parity suites, per-config bench lines (no CPU baseline).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TAG:-chk}
timeout 300 python scripts/stress_ring.py 2 > gpurun_out/stress_$T.log 2>&1; echo "exit $?" >> gpurun_out/stress_$T.log
for f in ${TESTS:-test_gpu_parity test_gpu_flags test_gpu_parity_large}; do
  timeout 1200 python -m pytest tests/$f.py -x -q --timeout 300 --timeout_method thread > gpurun_out/pytest_${T}_$f.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_${T}_$f.log
done
for c in ${CONFIGS:-c3 c4 c2 c5m c5r}; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio \
    > gpurun_out/bench_${T}_$c.json 2> gpurun_out/bench_${T}_$c.err
done
for c in ${CONFIGS:-c3 c4 c2 c5m c5r}; do
  python -c "import json; d=json.loads(open('gpurun_out/bench_${T}_$c.json').read().strip().splitlines()[-1]); print('$c', '%.4e'%d['value'], round(d['ms_per_step'],1),'ms')" 2>/dev/null || echo "$c FAILED"
done > gpurun_out/summary_$T.txt
for f in gpurun_out/pytest_${T}_*.log; do echo "$f: $(tail -n 2 $f | head -1)"; done >> gpurun_out/summary_$T.txt
cat gpurun_out/summary_$T.txt
