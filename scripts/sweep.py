"""Rate sweep over every BASELINE config and tracker / scheduler / build mode (1 GPU).

    python scripts/sweep.py [--particles-scale 1.0] [--out gpurun_out/sweep.json]

For each config the BASELINE history count is used (capped by --max-particles), 1 warm-up launch,
then `--reps` timed launches (CUDA events on the launching stream).  Reports segments/s,
histories/s and the segment count (which must agree between trackers: same walks).
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_13849_b200 as nt  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--max-particles", type=float, default=2e7)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "sweep.json"))
ap.add_argument("--configs", default="c1,c2,c3,c4,c5m,c5r")
a = ap.parse_args()

rows = []
for cfg in a.configs.split(","):
    spec, n_cfg = workloads.config(cfg)
    n = int(min(n_cfg, a.max_particles))
    if cfg == "c1":
        n = max(n, 1_000_000)          # C1's 1e4 histories take < 1 ms; time a larger batch
    variants = [("generic", "block", False), ("generic", "rounds", False), ("generic", "warp", False),
                ("generic", "history", False), ("generic", "dp", False), ("generic", "block", True),
                ("rect", "history", False)]
    for tracker, sched, pseudo in variants:
        m = nt.Model.from_spec(spec, device=0, pseudo_array=pseudo)
        if tracker == "rect" and not m.info["rect_specialisable"]:
            continue
        out = torch.zeros(m.out_len, dtype=torch.float64, device="cuda")
        m.track(min(n, 200_000), seed=99, out=out, tracker=tracker, scheduler=sched)
        torch.cuda.synchronize()
        t, seg = 0.0, 0
        for r in range(a.reps):
            out.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m.track(n, seed=workloads.SEED + r, out=out, tracker=tracker, scheduler=sched)
            e1.record()
            torch.cuda.synchronize()
            t += e0.elapsed_time(e1) / 1e3
            seg += m.unpack(out)["counters"]["segments"]
        row = {"config": spec["name"], "tracker": tracker, "scheduler": sched, "pseudo_array": pseudo,
               "histories": n, "segments": seg // a.reps, "segments_per_s": seg / t,
               "histories_per_s": n * a.reps / t, "ms_per_launch": 1e3 * t / a.reps,
               "depth": m.info["max_depth"], "n_cells": m.info["n_cells"],
               "device_bytes": m.info["device_bytes"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
        del m
os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(rows, f, indent=1)
