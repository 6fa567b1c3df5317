#!/bin/bash
# ncu --set full of each tracker/scheduler; raw + SASS-source CSVs are exported on the box
# (gpurun brings back <= 64 MiB), reports are kept only when KEEP=1.
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${TAG:-x}
LIST=${LIST:-"wq:k_track_wq:--scheduler%warp blk:k_track_event:--scheduler%block hist:k_track_generic:--scheduler%history rect:k_track_rect:--tracker%rect"}
for v in $LIST; do
  IFS=: read name kre args <<< "$v"
  args=${args//%/ }
  ncu --set full --clock-control none --import-source on -k regex:$kre -s 1 -c 1 -o /tmp/prof_${name}_$T \
    python bench.py --steps 1 --warmup 1 --particles ${NPART:-2e6} --no-cpu-baseline --no-e2e $args > gpurun_out/prof_${name}_$T.log 2>&1
  ncu -i /tmp/prof_${name}_$T.ncu-rep --page raw --csv > gpurun_out/prof_${name}_$T.raw.csv 2>/dev/null
  ncu -i /tmp/prof_${name}_$T.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_${name}_$T.sass.csv 2>/dev/null
  ncu -i /tmp/prof_${name}_$T.ncu-rep --page details > gpurun_out/prof_${name}_$T.details.txt 2>/dev/null
  if [ "${KEEP:-0}" = "1" ]; then cp /tmp/prof_${name}_$T.ncu-rep gpurun_out/; fi
done
echo done
