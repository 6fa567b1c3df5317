#!/bin/bash
# Round evidence: full GPU tests (incl. full-size C3), smoke, default bench line, ncu launch list of
# the same command, one ncu --set full capture of the dominant kernel in the bench configuration.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
R=${ROUND:-r01}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi_$R.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$R.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke_$R.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 > gpurun_out/pytest_gpu_$R.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_$R.log
timeout 900 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; echo "bench exit $?" >> gpurun_out/bench_$R.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$R.json 2> gpurun_out/bench_ref_$R.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ncu_launches_$R.csv \
    python bench.py --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/ncu_launches_bench_$R.log 2>&1
timeout 2400 ncu --set full --clock-control none --import-source on -k regex:k_track_event -s 3 -c 1 -o /tmp/prof_bench_$R \
    python bench.py --no-cpu-baseline --no-e2e --no-ratio --steps 1 --warmup 3 > gpurun_out/ncu_full_bench_$R.log 2>&1
ncu -i /tmp/prof_bench_$R.ncu-rep --page raw --csv > gpurun_out/ncu_full_$R.raw.csv 2>/dev/null
ncu -i /tmp/prof_bench_$R.ncu-rep --page details > gpurun_out/ncu_full_$R.details.txt 2>/dev/null
ncu -i /tmp/prof_bench_$R.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_full_$R.sass.csv 2>/dev/null
echo done
