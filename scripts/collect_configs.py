"""Collect the per-config bench lines and ncu DRAM-traffic captures of a profile pass
(scripts/gpu_r02_prof.sh) into profiles/: traffic.json (per-launch DRAM bytes of the tracking
kernel per workload), <round>_configs.json (the bench lines), and the BASELINE.md §4 table.

    python scripts/collect_configs.py --round r02 [--baseline]
"""
import argparse
import csv
import sys
import glob
import io
import json
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")
NAMES = {"c1": "C1 pincell", "c2": "C2 17x17 assembly", "c3": "C3 full-core PWR", "c4": "C4 hex microreactor",
         "c5m": "C5m deep nesting (mixed)", "c5r": "C5r deep nesting (rect-only)"}


def ncu_metrics(path):
    """{metric: value} of the single profiled launch in an `ncu --csv --metrics` log."""
    txt = open(path).read()
    start = txt.find('"ID"')
    if start < 0:
        return {}
    rows = list(csv.reader(io.StringIO(txt[start:])))
    h = rows[0]
    im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    out = {}
    for r in rows[1:]:
        if len(r) <= iv:
            continue
        v = float(r[iv].replace(",", ""))
        unit = r[iu]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "second": 1.0}.get(unit, 1.0)
        out[r[im]] = v * scale
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--round", default="r02")
    ap.add_argument("--baseline", action="store_true", help="rewrite BASELINE.md §4")
    ap.add_argument("--traffic-only", action="store_true",
                    help="update profiles/traffic.json from the ncu captures alone (before the bench lines exist)")
    a = ap.parse_args()
    import workloads
    names = {c: workloads.config(c)[0]["name"] for c in NAMES}
    lines, traffic = {}, {}
    tpath = os.path.join(PROF, "traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath))
    for c in NAMES:
        bp = os.path.join(OUT, f"bench_{c}_{a.round}.json")
        if os.path.exists(bp):
            js = [ln for ln in open(bp) if ln.startswith("{")]
            if js:
                lines[c] = json.loads(js[-1])
        tp = os.path.join(OUT, f"ncu_traffic_{c}_{a.round}.csv")
        if os.path.exists(tp):
            m = ncu_metrics(tp)
            if "dram__bytes_read.sum" in m:
                w = names[c]
                traffic[w] = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
                traffic[w + ".read"] = m["dram__bytes_read.sum"]
                traffic[w + ".write"] = m["dram__bytes_write.sum"]
                if c in lines:
                    traffic[w + ".thread_inst_per_segment"] = (
                        m.get("smsp__thread_inst_executed.sum", 0.0)
                        / max(lines[c]["value"] * lines[c]["ms_per_step"] / 1e3, 1.0))
    traffic["_doc"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the tracking kernel at each "
                       "workload's bench configuration (ncu --metrics, one launch after a warm-up), round " + a.round)
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)
    if a.traffic_only:
        return
    json.dump(lines, open(os.path.join(PROF, f"{a.round}_configs.json"), "w"), indent=1)
    rows = []
    for c, d in lines.items():
        rr = d.get("rect_ratio") or {}
        roof = d.get("roofline") or {}
        hbm = roof.get("hbm") or {}
        cpu = d.get("cpu_baseline") or {}
        n = d["config"]["histories_per_gpu_per_step"]
        segs = d["value"] * d["ms_per_step"] / 1e3
        rows.append(f"| {NAMES[c]} | 1 | {n:.0e} | {segs:.3e} | {d['value']:.3e} | {d['particles_per_s']:.3e} | "
                    + (f"{rr['generic_over_rect']:.2f} (ring/ring {rr['generic_ring_over_rect_ring']:.2f})" if rr else "n/a")
                    + f" | {roof.get('frac', 0) * 100:.2f} % | " + (f"{hbm['frac'] * 100:.4f} %" if hbm else "—")
                    + f" | {roof.get('binding', '—')} | "
                    + (f"{cpu['value']:.2e} ({cpu['cores']}); {cpu.get('value_1core', 0):.2e} (1)" if cpu else "—") + " |")
    table = "\n".join(rows)
    print(table)
    if a.baseline:
        p = os.path.join(ROOT, "BASELINE.md")
        s = open(p).read()
        head = s[:s.index("## 4.")]
        s4 = ("## 4. Results table (bench lines of this build, measured by the builder on 1 B200 via gpurun; " + a.round + ")\n\n"
              "Source: `python bench.py --config cN` (defaults: W = 3, K = 5, L2 flushed between steps), collected by "
              "`scripts/collect_configs.py` into `profiles/" + a.round + "_configs.json`.  fp64 frac = F_alg x "
              "segments/s / 37.2 TFLOP/s (derived peak); HBM frac = ncu DRAM bytes per launch / kernel time / "
              "measured HBM GB/s.  Multi-GPU rows: SCALE_rNN.json (driver).\n\n"
              "| Config | GPUs | particles | segments/step | segments/s | particles/s | generic / rect (best sched.) | "
              "fp64 frac | HBM frac | binding | oracle seg/s (cores) |\n"
              "|---|---|---|---|---|---|---|---|---|---|---|\n" + table + "\n")
        open(p, "w").write(head + s4)


if __name__ == "__main__":
    main()
