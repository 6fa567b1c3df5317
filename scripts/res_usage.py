"""Registers / stack / SASS size of the tracking kernels in libnestrack.so (quick check before GPU time)."""
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2406_13849_b200/libnestrack.so"
pat = sys.argv[2] if len(sys.argv) > 2 else r"f0.*(eventILi256ELb0ELb0ELb0E|genericILb0ELb0E|wqILb0ELb0E|rectILi2ELb0ELb0ELb0E)"
out = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
res, cur = {}, None
for ln in out.splitlines():
    m = re.match(r"\s*Function (\S+):", ln)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"REG:(\d+) STACK:(\d+)", ln)
    if m and cur:
        res[cur] = (int(m.group(1)), int(m.group(2)))
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
size, cur = {}, None
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1)
        continue
    if cur and re.match(r"\s+/\*[0-9a-f]{4,}\*/", ln):
        size[cur] = size.get(cur, 0) + 1
for k in sorted(res):
    if re.search(pat, k):
        print(f"{res[k][0]:4d} regs {res[k][1]:4d} B stack {size.get(k, 0):6d} SASS  {k}")
