"""Per-basic-block view of an ncu SASS-page export (`ncu -i X --page source --csv --print-source sass`).

    python scripts/sass_blocks.py <sass.csv> [--top 30]

Consecutive instructions with the same execution count form a block.  For each of the heaviest
blocks: address range, instruction count, share of warp instructions, active threads per
instruction and share of warp-stall samples; then the most-stalled single instructions and the
shared-memory wavefront excess (bank conflicts).
"""
import argparse
import csv

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("--top", type=int, default=30)
a = ap.parse_args()

rows = list(csv.reader(open(a.csv)))
kname = rows[0][1] if len(rows[0]) > 1 else ""
h = rows[1]
col = {k: h.index(k) for k in ("Address", "Source", "Instructions Executed", "Thread Instructions Executed",
                                "Warp Stall Sampling (All Samples)", "L1 Wavefronts Shared",
                                "L1 Wavefronts Shared Ideal") if k in h}
ins = []
for r in rows[2:]:
    if len(r) <= max(col.values()):
        continue
    try:
        addr = int(r[col["Address"]], 16)
    except ValueError:
        continue
    f = lambda k: float(r[col[k]] or 0) if k in col else 0.0
    ins.append((addr, r[col["Source"]].strip(), f("Instructions Executed"), f("Thread Instructions Executed"),
                f("Warp Stall Sampling (All Samples)"), f("L1 Wavefronts Shared"), f("L1 Wavefronts Shared Ideal")))
base = ins[0][0]
tot_e = sum(i[2] for i in ins) or 1.0
tot_w = sum(i[4] for i in ins) or 1.0
blocks, cur = [], None
for addr, src, e, t, w, _, _ in ins:
    if cur and cur["e"] == e and addr == cur["end"] + 16:
        cur["end"] = addr; cur["n"] += 1; cur["t"] += t; cur["w"] += w
    else:
        cur = {"start": addr, "end": addr, "e": e, "t": t, "w": w, "n": 1}
        blocks.append(cur)
print("kernel:", kname[:120])
print("warp instructions %.4e, thread instructions %.4e (%.1f per warp instruction), stall samples %.0f"
      % (tot_e, sum(i[3] for i in ins), sum(i[3] for i in ins) / tot_e, tot_w))
print("\n%-13s %4s %7s %6s %7s  first instruction" % ("offsets", "n", "inst%", "thr", "stall%"))
for b in sorted(blocks, key=lambda b: -b["e"] * b["n"])[:a.top]:
    first = next(i[1] for i in ins if i[0] == b["start"])
    print("%05x-%05x %4d %7.2f %6.1f %7.2f  %s" % (b["start"] - base, b["end"] - base, b["n"], 100 * b["e"] * b["n"] / tot_e,
                                                b["t"] / max(b["e"] * b["n"], 1), 100 * b["w"] / tot_w, first[:60]))
print("\nmost-stalled instructions:")
for addr, src, e, t, w, _, _ in sorted(ins, key=lambda i: -i[4])[:15]:
    print("%05x %7.2f%%  %s" % (addr - base, 100 * w / tot_w, src[:70]))
sw, si = sum(i[5] for i in ins), sum(i[6] for i in ins)
if si:
    print("\nshared-memory wavefronts %.3e, ideal %.3e: %.2fx (bank conflicts)" % (sw, si, sw / si))
