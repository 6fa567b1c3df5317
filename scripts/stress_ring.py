"""Stress the ring (ASYNC) scheduler with small batches (few blocks, many ring laps per block):
every config x ring variant x batch size, repeated; counters must be identical across repeats.
A hang here means a lost slot (the block never drains).  Run under `timeout`."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13849_b200 as nt  # noqa: E402
import workloads  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
t0 = time.time()
for cfg in ("c1", "c3", "c4", "c5m"):
    spec, _ = workloads.config(cfg)
    mesh = dict(spec, mesh={"lo": spec["source"]["lo"], "hi": spec["source"]["hi"], "shape": [8, 8, 4]})
    for sp in (spec, mesh):
        m = nt.Model.from_spec(sp, device=0)
        variants = [dict(scheduler="block"), dict(scheduler="dp")]
        if m.info["rect_specialisable"]:
            variants.append(dict(tracker="rect", scheduler="block"))
        for kw in variants:
            for n in (1, 37, 400, 3000, 20000):
                ref = None
                for r in range(reps):
                    res = m.track(n, seed=11, mesh=True if "mesh" in sp else None, **kw)
                    torch.cuda.synchronize()
                    c = m.unpack(res["out"])["counters"]
                    assert c["particles"] == n, (cfg, kw, n, c)
                    if ref is None:
                        ref = c
                    assert c == ref, (cfg, kw, n, r)
            print(f"{cfg}{' mesh' if 'mesh' in sp else ''} {kw}: ok ({time.time() - t0:.0f} s)", flush=True)
print("stress ok")
