#!/bin/bash
# A/B of tuning builds (tune/*.so) on the dispatch study (c2, c3): rates per method per build.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
timeout 900 python scripts/dispatch_study.py --configs ${CFGS:-c2,c3} --reps 2 --out gpurun_out/ab_main.json > gpurun_out/ab_main.log 2>&1
for lib in tune/*.so; do
  n=$(basename $lib .so)
  NESTRACK_LIB=$PWD/$lib timeout 900 python scripts/dispatch_study.py --configs ${CFGS:-c2,c3} --reps 2 --out gpurun_out/ab_$n.json > gpurun_out/ab_$n.log 2>&1
done
echo done
