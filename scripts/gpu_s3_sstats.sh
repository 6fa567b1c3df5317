cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
NESTRACK_LIB=$PWD/tune/libnestrack_sstats.so timeout 300 python scripts/safety_stats.py 1e6 > gpurun_out/sstats.txt 2>&1
for v in nosafe; do
 for c in c3 c4; do
  NESTRACK_LIB=$PWD/tune/libnestrack_$v.so timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/bench_${v}_$c.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/bench_${v}_$c.json').read().strip().splitlines()[-1]); print('$v $c', '%.4e'%d['value'])" >> gpurun_out/sstats.txt
 done
done
cat gpurun_out/sstats.txt
