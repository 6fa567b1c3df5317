"""Small tracking batches for compute-sanitizer (memcheck / racecheck / synccheck).

Runs C1 and C2 through every scheduler and the rect tracker with more histories than resident
ring slots (so slots are recycled), with tallies, flags and per-history outputs on.  Usage:

    compute-sanitizer --tool racecheck python scripts/sanitize.py --cfg c1 --n 200000
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2406_13849_b200 as nt  # noqa: E402
import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg", default="c1")
    ap.add_argument("--n", type=int, default=200000)
    ap.add_argument("--scheds", default="block,rounds,warp,history,dp,rect,rect-ring")
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    a = ap.parse_args()
    spec, _ = workloads.config(a.cfg)
    m = nt.Model.from_spec(spec, device=0)
    for s in a.scheds.split(","):
        tracker, sched = {"rect": ("rect", "history"), "rect-ring": ("rect", "block")}.get(s, ("generic", s))
        res = m.track(a.n, seed=7, pflags=True, per_history=True, scheduler=sched, tracker=tracker,
                      blocks_per_sm=a.blocks_per_sm)
        torch.cuda.synchronize()
        c = m.unpack(res["out"])["counters"]
        print(f"{a.cfg} {s}: n={a.n} launches={m.last_launch_count()} segments={c['segments']} "
              f"particles={c['particles']} lost={c['lost']} flagged={c['flagged']}", flush=True)
        assert c["particles"] == a.n and c["lost"] == 0


if __name__ == "__main__":
    main()
