"""Algorithmic fp64 flops per segment (F_alg) for every config, from the ORACLE's
distance-candidate evaluation counts (implementation-independent).  Writes profiles/falg.json.
Only calls oracle/ (a committed script, per the parity rules)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import workloads  # noqa: E402

out = {"_doc": "LINPACK-weighted fp64 flops per segment from oracle evaluation counts; weights "
               + json.dumps(oracle.EVAL_FLOPS) + "; sample = 20000 histories, seed 240613849"}
for name in workloads.CONFIGS:
    spec, _ = workloads.config(name)
    m = oracle.OracleModel.from_spec(spec)
    r = m.run(20000, seed=workloads.SEED)
    out[spec["name"]] = round(m.falg(r), 4)
    out[spec["name"] + ".segments_per_history"] = r["counters"]["segments"] / 20000
    print(spec["name"], out[spec["name"]], r["evals"])
with open(os.path.join(ROOT, "profiles", "falg.json"), "w") as f:
    json.dump(out, f, indent=1)
