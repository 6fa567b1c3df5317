"""Aggregate an ncu SASS source page (csv) by CUDA source line using nvdisasm -g line info.
usage: python scripts/ncu_lines.py <sass.csv> <nvdisasm -g output> <kernel mangled name> [topN]"""
import csv
import re
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
kern = sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# address -> (file, line, inlined-at chain top)
addr_line = {}
cur = None
inside = False
for ln in open(sys.argv[2]):
    if ln.startswith(".text.") or ln.startswith("\t.section\t.text."):
        inside = kern in ln
    m = re.match(r'\s*//## File "(.*)", line (\d+)(.*)', ln)
    if m and inside:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m and inside and cur:
        addr_line[int(m.group(1), 16)] = cur


def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0


agg = defaultdict(lambda: [0.0, 0.0, 0.0])
tot_s = tot_i = 0.0
base = int(data[0][ix["Address"]], 16)
for r in data:
    a = int(r[ix["Address"]], 16) - base
    key = addr_line.get(a, ("?", 0))
    s = f(r, "Warp Stall Sampling (All Samples)")
    i = f(r, "Instructions Executed")
    t = f(r, "Thread Instructions Executed")
    agg[key][0] += s
    agg[key][1] += i
    agg[key][2] += t
    tot_s += s
    tot_i += i
print(f"{'file:line':28s} {'stall%':>7s} {'inst%':>7s} {'thr/inst':>8s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]+':'+str(k[1]):28s} {100*v[0]/tot_s:7.2f} {100*v[1]/tot_i:7.2f} {v[2]/max(v[1],1):8.2f}")
