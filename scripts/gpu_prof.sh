#!/bin/bash
# ncu launch list + one full capture of the generic tracker; fp64 peak microbenchmark.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
./scripts/fp64_peak > gpurun_out/fp64_peak.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv \
    python bench.py --steps 2 --warmup 1 --particles 1e7 --no-cpu-baseline --no-e2e > gpurun_out/launches_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_track -s 1 -c 1 -o gpurun_out/prof_generic_r01 \
    python bench.py --steps 1 --warmup 1 --particles 2e6 --no-cpu-baseline --no-e2e > gpurun_out/prof_bench.log 2>&1
echo done
