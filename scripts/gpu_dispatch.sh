#!/bin/bash
# Dispatch study: rates of RTK / SP / DP / ST on every config, then one
# ncu --set full per method on C3 (i-fetch stalls = smsp__pcsamp_warps_issue_stalled_no_instructions,
# the metric the paper correlates with the DP slowdown).
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
T=${TAG:-disp}
timeout 1500 python scripts/dispatch_study.py --out gpurun_out/dispatch_$T.json > gpurun_out/dispatch_$T.log 2>&1
if [ "${PROF:-1}" = "1" ]; then
  TAG=$T LIST="sp:k_track_event:--scheduler%block dp:k_track_event:--scheduler%dp st:k_track_event:--pseudo-array rtk:k_track_rect:--tracker%rect" \
    NPART=${NPART:-2e6} timeout 2400 bash scripts/gpu_prof3.sh
fi
echo done
