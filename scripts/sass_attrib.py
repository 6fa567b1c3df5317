"""Attribute an ncu SASS-page export (scripts/gpu_prof3.sh *.sass.csv) to CUDA source lines.

    python scripts/sass_attrib.py <sass.csv> <kernel-substring> [--lib paper_2406_13849_b200/libnestrack.so]
                                  [--top 40] [--by inner|outer|chain]

The .so must be the binary that was profiled.  Instruction offsets come from the ncu export
(address - first address of the kernel) and are matched with `nvdisasm -gi` line info
(innermost source line, plus the chain of inlined-at call sites).  Prints warp-instruction
share, thread-instruction share, threads / instruction and stall-sample share per line.
"""
import argparse
import collections
import csv
import glob
import os
import re
import subprocess
import tempfile

ap = argparse.ArgumentParser()
ap.add_argument("csv")
ap.add_argument("kernel")
ap.add_argument("--lib", default=os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                              "paper_2406_13849_b200", "libnestrack.so"))
ap.add_argument("--top", type=int, default=40)
ap.add_argument("--by", default="outer", choices=["inner", "outer", "chain"])
a = ap.parse_args()

rows = list(csv.reader(open(a.csv)))
kname = rows[0][1] if len(rows[0]) > 1 else ""
h = rows[1]
iA, iE, iT, iS = (h.index(k) for k in ("Address", "Instructions Executed", "Thread Instructions Executed",
                                        "Warp Stall Sampling (All Samples)"))
prof = []
for r in rows[2:]:
    if len(r) <= iS:
        continue
    try:
        prof.append((int(r[iA], 16), float(r[iE] or 0), float(r[iT] or 0), float(r[iS] or 0)))
    except ValueError:
        pass
base = min(p[0] for p in prof)

tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", a.lib], cwd=tmp, check=True, capture_output=True)
lines = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    txt = subprocess.run(["nvdisasm", "-gi", "-c", cub], capture_output=True, text=True).stdout
    cur, info = None, None
    for ln in txt.splitlines():
        m = re.match(r"//-+ \.text\.(\S+) -+", ln)
        if m:
            cur = m.group(1) if a.kernel in m.group(1) else None
            continue
        if cur is None:
            continue
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', ln)
        if m:
            chain = [(os.path.basename(m.group(1)), int(m.group(2)))]
            for f, l in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3)):
                chain.append((os.path.basename(f), int(l)))
            info = chain
            continue
        m = re.search(r"/\*([0-9a-f]{4,})\*/", ln)
        if m and info is not None:
            lines[(cur, int(m.group(1), 16))] = info
    if lines:
        break
funcs = {k[0] for k in lines}
assert len(funcs) >= 1, "kernel not found in " + a.lib
fn = sorted(funcs, key=len)[0]
print("kernel:", fn, "| ncu:", kname[:100])

src_cache = {}


def src(f, l):
    if f not in src_cache:
        p = glob.glob(os.path.join(os.path.dirname(a.lib), "csrc", f))
        src_cache[f] = open(p[0]).read().splitlines() if p else []
    s = src_cache[f]
    return s[l - 1].strip()[:70] if 0 < l <= len(s) else ""


agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
tot = [0.0, 0.0, 0.0]
for addr, e, t, s in prof:
    chain = lines.get((fn, addr - base))
    if chain is None:
        key = ("?", 0)
    elif a.by == "inner":
        key = chain[0]
    elif a.by == "outer":
        key = chain[-1]
    else:
        key = tuple(chain)
    v = agg[key]
    v[0] += e; v[1] += t; v[2] += s
    tot[0] += e; tot[1] += t; tot[2] += s
print("warp inst %.3e  thread inst %.3e  thr/inst %.1f" % (tot[0], tot[1], tot[1] / max(tot[0], 1)))
print("%-28s %6s %6s %5s %6s  %s" % ("line", "warp%", "thr%", "t/i", "stall%", "source"))
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:a.top]:
    head = k[0] if a.by != "chain" else k[0]
    f, l = head if isinstance(head, tuple) else k
    label = "%s:%d" % (f, l) if a.by != "chain" else " <- ".join("%s:%d" % x for x in k)[:60]
    print("%-28s %6.2f %6.2f %5.1f %6.2f  %s" % (label[:28], 100 * v[0] / tot[0], 100 * v[1] / tot[1],
                                                 v[1] / max(v[0], 1), 100 * v[2] / max(tot[2], 1), src(f, l)))
