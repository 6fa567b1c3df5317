#!/bin/bash
# One ncu --set full capture of the default tracker at a reduced batch (2e6 C3 histories) with the
# SASS page exported for scripts/sass_attrib.py, plus a short bench line for context.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${TAG:-attrib}
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-ratio ${EXTRA} > gpurun_out/bench_$T.json 2> gpurun_out/bench_$T.err
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_track_event} -s 1 -c 1 -o /tmp/prof_$T \
    python bench.py --steps 1 --warmup 1 --particles 1e7 --no-cpu-baseline --no-e2e --no-ratio ${EXTRA} > gpurun_out/prof_$T.log 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_$T.raw.csv 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$T.sass.csv 2>/dev/null
echo done
