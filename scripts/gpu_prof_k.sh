#!/bin/bash
# usage: KREGEX=... TAG=... EXTRA="bench args" bash scripts/gpu_prof_k.sh
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
ncu --set full --clock-control none --import-source on -k regex:${KREGEX} -s 1 -c 1 -o gpurun_out/prof_${TAG} \
    python bench.py --steps 1 --warmup 1 --particles 2e6 --no-cpu-baseline --no-e2e ${EXTRA} > gpurun_out/prof_${TAG}.log 2>&1
echo done
