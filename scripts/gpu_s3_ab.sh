#!/bin/bash
# A/B of tuning builds (tune/libnestrack_<v>.so; "base" = in-tree): bench lines per config, optional
# safety-skip statistics for *stats builds.  No parity here: run gpu_s3_check.sh on the winner.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TAG:-ab}
: > gpurun_out/ab_$T.txt
for v in ${STATS}; do
  NESTRACK_LIB=$PWD/tune/libnestrack_$v.so timeout 300 python scripts/safety_stats.py 1e6 ${CONFIGS// /,} >> gpurun_out/ab_$T.txt 2>&1
done
for v in ${VARIANTS}; do
  if [ "$v" = base ]; then unset NESTRACK_LIB; else export NESTRACK_LIB=$PWD/tune/libnestrack_$v.so; fi
  for c in ${CONFIGS:-c3 c4}; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/ab_${T}_${v}_$c.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/ab_${T}_${v}_$c.json').read().strip().splitlines()[-1]); print('$v $c', '%.4e'%d['value'])" >> gpurun_out/ab_$T.txt 2>&1 || echo "$v $c FAILED" >> gpurun_out/ab_$T.txt
  done
done
unset NESTRACK_LIB
cat gpurun_out/ab_$T.txt
