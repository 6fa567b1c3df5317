"""Safety-skip diagnostics (tuning build with -DNT_SAFETY_STATS, selected by NESTRACK_LIB): per config,
the fraction of MOVEs with upper levels that were deferred to the U ring, and why."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_13849_b200 as nt  # noqa: E402
import workloads  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000000
for cfg in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["c2", "c3", "c4", "c5m", "c5r"]):
    spec, _ = workloads.config(cfg)
    m = nt.Model.from_spec(spec, device=0)
    res = m.track(n, seed=3)
    torch.cuda.synchronize()
    c = m.unpack(res["out"])["counters"]
    mv, de, inv, u = c["cross_l4"], c["cross_l5"], c["cross_l6"], c["cross_l7"]
    print(f"{cfg}: segments {c['segments']}  mode-0 moves with upper levels {mv} ({mv / c['segments']:.3f} of segments)  "
          f"deferred {de} ({de / max(mv, 1):.3f})  no covering bound {inv} ({inv / max(mv, 1):.3f})  U moves {u}")
