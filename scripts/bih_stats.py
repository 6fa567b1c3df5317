"""Debug: BIH traversal counters per config (tuning build tune/lib_bihstats.so)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["NESTRACK_LIB"] = os.path.join(ROOT, "tune", "lib_bihstats.so")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2406_13849_b200 as nt  # noqa: E402
import workloads  # noqa: E402

L = nt.lib()
L.nt_debug_bih_stats.argtypes = [C.c_int32, C.c_void_p, C.c_int32]
for cfg in ["c3", "c4", "c2"]:
    for pseudo in (False, True):
        spec, _ = workloads.config(cfg)
        m = nt.Model.from_spec(spec, device=0, pseudo_array=pseudo)
        fset = 0 if m.L and spec and True else 0
        buf = np.zeros(4, dtype=np.uint64)
        for fs in (0, 7):
            L.nt_debug_bih_stats(fs, buf.ctypes.data_as(C.c_void_p), 1)
        res = m.track(200000, seed=1)
        torch.cuda.synchronize()
        tot = np.zeros(4)
        for fs in (0, 7):
            L.nt_debug_bih_stats(fs, buf.ctypes.data_as(C.c_void_p), 0)
            tot += buf
        seg = m.unpack(res["out"])["counters"]["segments"]
        print(cfg, "pseudo" if pseudo else "generic", "calls/seg %.2f nodes/call %.2f cells/call %.2f" %
              (tot[0] / seg, tot[1] / max(tot[0], 1), tot[2] / max(tot[0], 1)))
