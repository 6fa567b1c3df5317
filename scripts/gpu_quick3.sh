#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_q3.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q3.log
for c in c3 c4 c2; do
  for b in 256 192; do
    timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --config $c --block-dim $b > gpurun_out/bq3_${c}_$b.json 2>&1
  done
done
echo done
