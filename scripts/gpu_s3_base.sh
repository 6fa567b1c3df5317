#!/bin/bash
# Session baseline: smoke, GPU parity suite, default bench line, one ncu --set full capture of the
# C3 ring kernel with the SASS page (for scripts/sass_attrib.py).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TAG:-s3base}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_$T.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$T.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 600 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/bench_c4_$T.json 2> gpurun_out/bench_c4_$T.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_track_event -s 1 -c 1 -o /tmp/prof_$T \
    python bench.py --steps 1 --warmup 1 --particles 1e7 --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/prof_$T.log 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_$T.raw.csv 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$T.sass.csv 2>/dev/null
cp paper_2406_13849_b200/libnestrack.so gpurun_out/libnestrack_$T.so
if [ -z "$SKIP_TESTS" ]; then
for f in test_gpu_parity test_gpu_flags test_gpu_parity_large test_distributed_gpu; do
  timeout 1500 python -m pytest tests/$f.py -q --timeout 400 --timeout_method thread > gpurun_out/pytest_${T}_$f.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_${T}_$f.log
done
fi
echo done
