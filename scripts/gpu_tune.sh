#!/bin/bash
# bench each tune/*.so (NESTRACK_LIB) with the given scheduler list
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for lib in tune/*.so; do
  for sch in ${SCHEDS:-block history}; do
    name=$(basename $lib .so)_$sch
    NESTRACK_LIB=$PWD/$lib timeout 600 python bench.py --steps 2 --warmup 1 --particles ${NPART:-1e7} --no-cpu-baseline --no-e2e --no-ratio --scheduler $sch ${EXTRA} > gpurun_out/tune_$name.log 2>&1
  done
done
for f in gpurun_out/tune_*.log; do python -c "
import json,sys
try:
  d=json.loads(open('$f').readline()); print('%-40s %.3e seg/s'%('$f', d['value']))
except Exception as e: print('$f ERR')"; done > gpurun_out/tune_summary.txt
