#!/bin/bash
# Round-2 profile pass: per-config bench lines, DRAM traffic per config (ncu), one ncu --set full
# capture of the C3 ring kernel (+ SASS source page) and one of the C4 ring kernel.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
R=${ROUND:-r02}
# DRAM traffic per config first (ncu, one launch after a warm-up), so that the bench lines below
# carry this build's HBM fraction
for c in ${CONFIGS:-c1 c2 c3 c4 c5m c5r}; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum,smsp__thread_inst_executed.sum \
    --clock-control none -k regex:k_track_event -s 1 -c 1 --csv \
    python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-ratio --no-cpu-baseline \
    > gpurun_out/ncu_traffic_${c}_$R.csv 2> gpurun_out/ncu_traffic_${c}_$R.err
done
python scripts/collect_configs.py --round $R --traffic-only > /dev/null 2>&1
for c in ${CONFIGS:-c1 c2 c3 c4 c5m c5r}; do
  timeout 900 python bench.py --config $c --cpu-seconds 8 > gpurun_out/bench_${c}_$R.json 2> gpurun_out/bench_${c}_$R.err
done
# DRAM traffic vs batch size (is the write traffic per launch or per history?)
for n in 1e6 1e7; do
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_srcunit_tex_op_red.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_st.sum,l1tex__t_bytes_pipe_lsu_mem_local_op_ld.sum \
    --clock-control none -k regex:k_track_event -s 1 -c 1 --csv \
    python bench.py --particles $n --steps 1 --warmup 1 --no-e2e --no-ratio --no-cpu-baseline \
    > gpurun_out/ncu_traffic_c3_n${n}_$R.csv 2> gpurun_out/ncu_traffic_c3_n${n}_$R.err
done
if [ -z "$SKIP_FULL" ]; then
for c in c3 c4; do
  timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_track_event -s 3 -c 1 -o /tmp/prof_${c}_$R \
    python bench.py --config $c --no-cpu-baseline --no-e2e --no-ratio --steps 1 --warmup 3 > gpurun_out/ncu_full_${c}_$R.log 2>&1
  ncu -i /tmp/prof_${c}_$R.ncu-rep --page raw --csv > gpurun_out/ncu_full_${c}_$R.raw.csv 2>/dev/null
  ncu -i /tmp/prof_${c}_$R.ncu-rep --page details > gpurun_out/ncu_full_${c}_$R.details.txt 2>/dev/null
  ncu -i /tmp/prof_${c}_$R.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_full_${c}_$R.sass.csv 2>/dev/null
done
cp paper_2406_13849_b200/libnestrack.so gpurun_out/libnestrack_$R.so
fi
[ -n "$SKIP_SAN" ] || for s in rounds dp rect-ring; do
  timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python scripts/sanitize.py --cfg c1 --n 200000 --scheds $s \
    > gpurun_out/racecheck_${R}_c1_$s.log 2>&1; echo "exit $?" >> gpurun_out/racecheck_${R}_c1_$s.log
done
echo done
