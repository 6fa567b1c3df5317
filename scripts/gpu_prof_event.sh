#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
TAG=${TAG:-r01}
ncu --set full --clock-control none --import-source on -k regex:k_track_event -s 1 -c 1 -o gpurun_out/prof_event_$TAG \
    python bench.py --steps 1 --warmup 1 --particles 2e6 --no-cpu-baseline --no-e2e > gpurun_out/prof_event.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_track_rect -s 1 -c 1 -o gpurun_out/prof_rect_$TAG \
    python bench.py --steps 1 --warmup 1 --particles 2e6 --no-cpu-baseline --no-e2e --tracker rect > gpurun_out/prof_rect.log 2>&1
echo done
