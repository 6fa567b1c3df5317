#!/bin/bash
# Round-2 final evidence (third session): stress, smoke, every GPU test file, default bench line,
# reference arm, ncu launch list, per-config profile pass (scripts/gpu_r02_prof.sh), sanitizers on
# the kernels changed this session (f7 recomputed frames / 384 slots, deep-model tier), dispatch study.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
R=${ROUND:-r02}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$R.txt 2>&1
timeout 400 python scripts/stress_ring.py 5 > gpurun_out/stress_$R.log 2>&1; echo "exit $?" >> gpurun_out/stress_$R.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$R.log
for f in test_gpu_parity test_gpu_flags test_gpu_parity_large test_distributed_gpu; do
  timeout 1200 python -m pytest tests/$f.py -q --timeout 300 --timeout_method thread > gpurun_out/pytest_${R}_$f.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_${R}_$f.log
done
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench exit $?" >> gpurun_out/bench_$R.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_$R.csv \
    python bench.py --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/ncu_launches_bench_$R.log 2>&1
ROUND=$R SKIP_SAN=1 bash scripts/gpu_r02_prof.sh
[ -n "$SKIP_SAN" ] || for c in c4 c5r; do
  for t in memcheck synccheck; do
    timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py --cfg $c --n 200000 --scheds block \
      > gpurun_out/sanitize_${t}_${c}_$R.log 2>&1; echo "exit $?" >> gpurun_out/sanitize_${t}_${c}_$R.log
  done
done
timeout 1500 python scripts/dispatch_study.py --configs ${DISPATCH:-c1,c2,c3,c5r,c4,c5m} --out gpurun_out/dispatch_$R.json > gpurun_out/dispatch_$R.log 2>&1
echo done
