#!/bin/bash
# Round-1 widening check: full GPU tests, default bench, mesh-tally bench (119x119x30), block 128,
# dispatch study (ST with direction-ordered BIH search).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1800 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_gpu_next.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_next.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_next.json 2> gpurun_out/bench_next.err
timeout 900 python bench.py --no-cpu-baseline --mesh 119x119x30 > gpurun_out/bench_mesh.json 2> gpurun_out/bench_mesh.err
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --block-dim 128 > gpurun_out/bench_b128.json 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 > gpurun_out/bench_b256.json 2>&1
timeout 1500 python scripts/dispatch_study.py --out gpurun_out/dispatch_next.json > gpurun_out/dispatch_next.log 2>&1
echo done
