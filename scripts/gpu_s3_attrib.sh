#!/bin/bash
# ncu --set full of the ring kernel (1e7 histories of CONFIG) with the SASS page, plus the .so profiled
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
mkdir -p gpurun_out
T=${TAG:-attrib}; C=${CONFIG:-c3}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-k_track_event} -s 1 -c 1 -o /tmp/prof_$T \
    python bench.py --config $C --steps 1 --warmup 1 --particles ${NP:-1e7} --no-cpu-baseline --no-e2e --no-ratio > gpurun_out/prof_$T.log 2>&1
ncu -i /tmp/prof_$T.ncu-rep --page raw --csv > gpurun_out/ncu_$T.raw.csv 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page details > gpurun_out/ncu_$T.details.txt 2>/dev/null
ncu -i /tmp/prof_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_$T.sass.csv 2>/dev/null
cp ${NESTRACK_LIB:-paper_2406_13849_b200/libnestrack.so} gpurun_out/libnestrack_$T.so
echo done
