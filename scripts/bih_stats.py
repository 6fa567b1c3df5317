"""Debug: BIH traversal counters per config (tuning build tune/lib_bihstats.so, -DNT_BIH_STATS):
calls per segment, node visits and cell tests per call, the maxima and the log2 histogram of cell
tests per call."""
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
for cfg in (sys.argv[1].split(",") if len(sys.argv) > 1 else ["c3", "c4", "c2"]):
    for pseudo in (False, True):
        spec, _ = workloads.config(cfg)
        m = nt.Model.from_spec(spec, device=0, pseudo_array=pseudo)
        buf = np.zeros(16, dtype=np.uint64)
        for fs in (0, 7):
            L.nt_debug_bih_stats(fs, buf.ctypes.data_as(C.c_void_p), 1)
        res = m.track(200000, seed=1)
        torch.cuda.synchronize()
        tot = np.zeros(16)
        for fs in (0, 7):
            L.nt_debug_bih_stats(fs, buf.ctypes.data_as(C.c_void_p), 0)
            tot[:4] += buf[:4]
            tot[4:6] = np.maximum(tot[4:6], buf[4:6])
            tot[6:] += buf[6:]
        seg = m.unpack(res["out"])["counters"]["segments"]
        print(cfg, "pseudo" if pseudo else "generic",
              "calls/seg %.2f nodes/call %.2f cells/call %.2f max cells %d max nodes %d" %
              (tot[0] / seg, tot[1] / max(tot[0], 1), tot[2] / max(tot[0], 1), tot[4], tot[5]),
              "hist(cells: 0,1,2-3,4-7,..):", tot[6:].astype(int).tolist(), flush=True)
