#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 900 > gpurun_out/pytest_q2.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q2.log
for c in c3 c4 c2; do
  timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-ratio --particles 2e7 --config $c > gpurun_out/bq2_$c.json 2>&1
done
echo done
