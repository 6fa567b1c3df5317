"""Dispatch-strategy study on one B200 (§4 methods P:683-863, Table 2
P:1054-1080): the same walks tracked with

  RTK  rect-specialised tracker (Alg. 9-10)            tracker="rect"
  SP   switch on the universe kind (default kernel)     scheduler="block"
  DP   virtual tracker objects (nt_run.flags NT_DP)     scheduler="dp"
  ST   pseudo-array universes, all CSG + BIH            pseudo_array=True

and reported as segments/s and as a fraction of the RTK rate (the paper's Table 2 metric), with
the segment counts that prove the walks are the same.  All four share the ring (block-queue)
scheduler; RTK-H is the rect-specialised tracker's own history-based kernel.

    python scripts/dispatch_study.py [--configs c2,c3,c5r,c4,c5m] [--reps 3] [--out gpurun_out/dispatch.json]
"""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2406_13849_b200 as nt  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c2,c3,c5r,c4,c5m")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--max-particles", type=float, default=2e7)
ap.add_argument("--st-particles", type=float, default=2e6, help="ST runs are slower; smaller batch")
ap.add_argument("--min-particles", type=float, default=1e7,
                help="rate batches at least this large (C1's BASELINE batch, 1e4, is launch-latency bound)")
ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "dispatch.json"))
a = ap.parse_args()

VARIANTS = [("RTK", dict(tracker="rect", scheduler="block"), False),
            ("RTK-H", dict(tracker="rect", scheduler="history"), False),
            ("SP", dict(scheduler="block"), False),
            ("DP", dict(scheduler="dp"), False),
            ("ST", dict(scheduler="block"), True)]

rows = []
for cfg in a.configs.split(","):
    spec, n_cfg = workloads.config(cfg)
    models = {}
    for name, kw, pseudo in VARIANTS:
        if pseudo not in models:
            models[pseudo] = nt.Model.from_spec(spec, device=0, pseudo_array=pseudo)
        m = models[pseudo]
        if kw.get("tracker") == "rect" and not m.info["rect_specialisable"]:
            continue
        n = int(a.st_particles if pseudo else min(max(n_cfg, a.min_particles), a.max_particles))
        out = torch.zeros(m.out_len, dtype=torch.float64, device="cuda")
        m.track(min(n, 100_000), seed=99, out=out, **kw)        # warm-up (module load, DP objects)
        torch.cuda.synchronize()
        rates, seg = [], None
        for r in range(a.reps):
            out.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            m.track(n, seed=workloads.SEED + r, out=out, **kw)
            e1.record()
            torch.cuda.synchronize()
            s = m.unpack(out)["counters"]["segments"]
            seg = s if seg is None else seg
            rates.append(s / (e0.elapsed_time(e1) / 1e3))
        row = {"config": spec["name"], "method": name, "histories": n, "segments_rep0": seg,
               "segments_per_s": statistics.median(rates),
               "cv": statistics.pstdev(rates) / statistics.mean(rates) if len(rates) > 1 else 0.0}
        rows.append(row)
        print(json.dumps(row), flush=True)
    # fraction of the RTK rate (only where RTK runs); ST at a smaller batch is rate-comparable
    rtk = next((r["segments_per_s"] for r in rows if r["config"] == spec["name"] and r["method"] == "RTK"), None)
    for r in rows:
        if r["config"] == spec["name"]:
            r["fraction_of_rtk"] = r["segments_per_s"] / rtk if rtk else None
    del models

os.makedirs(os.path.dirname(a.out), exist_ok=True)
with open(a.out, "w") as f:
    json.dump(rows, f, indent=1)
print("\n| config | method | segments/s | % of RTK | cv |")
print("|---|---|---|---|---|")
for r in rows:
    fr = "%.1f" % (100 * r["fraction_of_rtk"]) if r.get("fraction_of_rtk") else "—"
    print("| %s | %s | %.3g | %s | %.3f |" % (r["config"], r["method"], r["segments_per_s"], fr, r["cv"]))
