#!/bin/bash
# A/B: GPU parity suite on the in-tree build, then the default bench line for the in-tree build and
# every tune/*.so (NESTRACK_LIB), block 256 and 192.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${TAG:-ab}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_$T.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_$T.log
B="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio ${EXTRA}"
for bd in ${BDS:-256 192}; do
  timeout 300 python bench.py $B --block-dim $bd > gpurun_out/bench_${T}_main_$bd.json 2>&1
  for lib in tune/*.so; do
    n=$(basename $lib .so)
    NESTRACK_LIB=$PWD/$lib timeout 300 python bench.py $B --block-dim $bd > gpurun_out/bench_${T}_${n}_$bd.json 2>&1
  done
done
echo done
