"""One-screen summary of ncu reports: time, occupancy, issue, divergence, stall breakdown."""
import csv
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "time"), ("launch__registers_per_thread", "regs"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("smsp__thread_inst_executed_per_inst_executed.ratio", "thr/inst"),
        ("smsp__inst_executed.sum", "inst"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64pipe%"),
        ("dram__bytes_read.sum", "dram_rd"), ("dram__bytes_write.sum", "dram_wr")]


def load(path):
    if path.endswith(".csv"):
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    return {h: (v, u) for h, v, u in zip(rows[0], rows[2], rows[1])}


for p in sys.argv[1:]:
    d = load(p)
    print("==", p)
    print("  " + "  ".join(f"{lab}={d[k][0]}{d[k][1] if d[k][1] not in ('', 'inst') else ''}" for k, lab in KEYS if k in d))
    ks = [k for k in d if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st = sorted(((float(d[k][0] or 0), k) for k in ks), reverse=True)[:7]
    print("  stalls/issue: " + ", ".join(f"{k[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={v:.2f}" for v, k in st))
