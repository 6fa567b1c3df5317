#!/bin/bash
# Round-end evidence: everything the judge reads under profiles/ (bench lines, reference arm,
# launch list, ncu full capture + SASS page, sweep, dispatch study, mesh bench).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
R=${ROUND:-r01}
bash scripts/gpu_round_evidence.sh
timeout 900 python bench.py --no-cpu-baseline --mesh 119x119x30 > gpurun_out/bench_mesh_$R.json 2> gpurun_out/bench_mesh_$R.err
timeout 1500 python scripts/dispatch_study.py --out gpurun_out/dispatch_$R.json > gpurun_out/dispatch_$R.log 2>&1
timeout 1200 python scripts/sweep.py --configs c1,c2,c3,c4,c5m,c5r --reps 2 --out gpurun_out/sweep_$R.json > gpurun_out/sweep_$R.log 2>&1
echo done
