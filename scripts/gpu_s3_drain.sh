#!/bin/bash
# Launch-size dependence of the C3 rate (fixed per-launch drain cost?)
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
for n in 2.5e7 5e7 1e8 2e8 4e8; do
  timeout 900 python bench.py --particles $n --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio 2>/dev/null | tail -1 > gpurun_out/drain_$n.json
  python -c "import json; d=json.load(open('gpurun_out/drain_$n.json')); print('$n', '%.4e'%d['value'], round(d['ms_per_step'],1))"
done
