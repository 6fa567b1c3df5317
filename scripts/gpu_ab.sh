#!/bin/bash
# A/B of tuning builds: parity subset + C3/C4 bench per variant (NESTRACK_LIB selects the .so).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
TAG=${TAG:-ab}
for v in base ${VARIANTS}; do
  if [ "$v" = base ]; then unset NESTRACK_LIB; else export NESTRACK_LIB=$PWD/tune/libnestrack_$v.so; fi
  timeout 240 python scripts/stress_ring.py 2 > gpurun_out/${TAG}_${v}_stress.log 2>&1
  if [ $? -ne 0 ]; then echo "stress failed: skipping $v" >> gpurun_out/${TAG}_${v}_stress.log; continue; fi
  timeout 600 python -m pytest tests/test_gpu_parity.py -x -q --timeout 300 --timeout_method thread \
    -k "config_trace_parity or rect_tracker or mesh_tally or instance or fission_bank" > gpurun_out/${TAG}_${v}_pytest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${TAG}_${v}_pytest.log
  for c in ${CONFIGS:-c3 c4}; do
    timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio \
      > gpurun_out/${TAG}_${v}_$c.json 2> gpurun_out/${TAG}_${v}_$c.err
  done
done
unset NESTRACK_LIB
for v in base ${VARIANTS}; do for c in ${CONFIGS:-c3 c4}; do
  python -c "import json,sys; d=json.load(open('gpurun_out/${TAG}_${v}_$c.json')); print('$v $c', round(d['value']/1e9,3), 'Gseg/s', round(d['ms_per_step'],1), 'ms')" 2>/dev/null || echo "$v $c FAILED"
done; grep -h "passed\|failed" gpurun_out/${TAG}_${v}_pytest.log | tail -1; done > gpurun_out/${TAG}_summary.txt
cat gpurun_out/${TAG}_summary.txt
