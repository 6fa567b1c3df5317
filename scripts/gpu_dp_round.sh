#!/bin/bash
# DP dispatch: parity tests, dispatch study, bench-config full ncu capture, per-method profiles.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python -m pytest tests -m gpu -q -x -k "dp or pseudo_hex" > gpurun_out/pytest_dp.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_dp.log
TAG=disp PROF=0 bash scripts/gpu_dispatch.sh
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_track_event -s 3 -c 1 -o /tmp/prof_bench_r01 \
    python bench.py --no-cpu-baseline --no-e2e --no-ratio --steps 1 --warmup 3 > gpurun_out/ncu_full_bench_r01.log 2>&1
ncu -i /tmp/prof_bench_r01.ncu-rep --page raw --csv > gpurun_out/ncu_full_r01.raw.csv 2>/dev/null
ncu -i /tmp/prof_bench_r01.ncu-rep --page details > gpurun_out/ncu_full_r01.details.txt 2>/dev/null
ncu -i /tmp/prof_bench_r01.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_full_r01.sass.csv 2>/dev/null
TAG=disp LIST="dp:k_track_event:--scheduler%dp st:k_track_event:--pseudo-array" NPART=2e6 timeout 2400 bash scripts/gpu_prof3.sh
echo done
