cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
B="--steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio --particles 2e7"
for t in "--scheduler history" "--tracker rect"; do
  n=$(echo $t | tr -d ' -')
  timeout 300 python bench.py $B $t > gpurun_out/bench_v10x_main_$n.json 2>&1
  NESTRACK_LIB=$PWD/tune/v8.so timeout 300 python bench.py $B $t > gpurun_out/bench_v10x_v8_$n.json 2>&1
done
