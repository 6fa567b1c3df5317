#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_c2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_c2.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 900 python bench.py --no-cpu-baseline --no-ratio --mesh 119x119x30 > gpurun_out/bench_mesh_c2.json 2> gpurun_out/bench_mesh_c2.err
timeout 1500 python scripts/dispatch_study.py --out gpurun_out/dispatch_c2.json > gpurun_out/dispatch_c2.log 2>&1
timeout 900 python scripts/sweep.py --configs c1,c2,c3,c4,c5m,c5r --reps 2 --out gpurun_out/sweep_c2.json > gpurun_out/sweep_c2.log 2>&1
echo done
