#!/bin/bash
for f in warp block history rect; do python -c "
import json,sys
try:
  d=json.loads(open('gpurun_out/bench_$f.log').readline()); print('%-8s %.3e seg/s  %7.1f ms  seg=%d'%('$f',d['value'], d['ms_per_step'], d['counters_last_step']['segments']))
except Exception as e: print('$f', 'ERR', open('gpurun_out/bench_$f.log').read()[-300:])"; done
