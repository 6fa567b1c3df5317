"""Benchmark: track segments/s on the full-core PWR (C3) at N GPUs (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nestrack|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

A step = one pass of the whole hot path (birth -> descend -> segment loop -> tally flush, plus
the one all-reduce of the packed tallies when N > 1) over one batch of C3 histories generated on
the device from (seed, pid).  Weak scaling: each rank tracks `--particles` histories per step
(default 1e8, the BASELINE C3 batch) from its own contiguous pid range.  Rank 0 prints one JSON
line.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "track segments/s, full-core PWR at 1/2/4/8 B200; ratio vs rectilinear tracker"
UNIT = "segments/s"
PROFILES = os.path.join(ROOT, "profiles")


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nestrack", choices=["nestrack", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--particles", type=float, default=None, help="histories per GPU per step")
    ap.add_argument("--tracker", default="generic", choices=["generic", "rect"])
    ap.add_argument("--scheduler", default="block", choices=["block", "rounds", "warp", "history", "dp", "dp-rounds"])
    ap.add_argument("--pseudo-array", action="store_true")
    ap.add_argument("--block-dim", type=int, default=0)
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-ratio", action="store_true", help="skip the rect-tracker comparison run")
    ap.add_argument("--mesh", default=None, help="superimposed mesh tally NXxNYxNZ over the config's "
                    "source box (NEXT-2; the paper's active-cycle mesh is 119x119x30)")
    return ap.parse_args()


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """Samples SM clocks and throttle reasons (NVML) during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
        except Exception:
            return self

        def loop():
            while not self._stop.is_set():
                try:
                    self.samples.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
                    r = pynvml.nvmlDeviceGetCurrentClocksEventReasons(h)
                    for bit, name in self.REASONS.items():
                        if r & bit and name != "gpu_idle":
                            self.reasons.add(name)
                except Exception:
                    pass
                time.sleep(0.1)

        self._t = threading.Thread(target=loop, daemon=True)
        self._t.start()
        return self

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join()
        s = sorted(self.samples)
        return {"sm_mhz": s[len(s) // 2] if s else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(s)}


def _load_json(name):
    p = os.path.join(PROFILES, name)
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def _measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return None


def _traffic_key(name, a, mesh_shape):
    """profiles/traffic.json holds one ncu capture per (workload, variant) that was profiled."""
    k = name
    if a.tracker != "generic":
        k += ".rect"
    elif a.scheduler != "block":
        k += "." + a.scheduler
    if a.pseudo_array:
        k += ".pseudo"
    if mesh_shape:
        k += ".mesh" + "x".join(map(str, mesh_shape))
    return k


def fp64_peak_tflops(sm_max_mhz: float | None) -> float:
    """fp64 FMA peak derived from unit counts: 148 SMs x 64 FP64 lanes x
    2 flop/FMA x max SM clock (1965 MHz) = 37.2 TFLOP/s."""
    mhz = sm_max_mhz or 1965.0
    return 148 * 64 * 2 * mhz * 1e6 / 1e12


def cpu_baseline(spec, seed: int, budget_s: float):
    """The oracle as it stands, on this host's cores, on a bounded sample of the workload."""
    import oracle
    om = oracle.OracleModel.from_spec(spec)
    cores = len(os.sched_getaffinity(0))
    n = 2000
    t = time.perf_counter()
    r = om.run(n, seed=seed, threads=cores)
    dt = time.perf_counter() - t
    # scale the sample to ~budget_s of CPU work
    n2 = int(min(max(n * budget_s / max(dt, 1e-3), n), 5_000_000))
    t = time.perf_counter()
    r = om.run(n2, seed=seed, pid_begin=10_000_000, threads=cores)
    dt = time.perf_counter() - t
    seg = r["counters"]["segments"]
    # the same oracle on one core, on a smaller sample (~budget/3 s)
    n1 = int(max(200, n2 * (budget_s / 3.0) / max(dt * cores, 1e-3)))
    t = time.perf_counter()
    r1 = om.run(n1, seed=seed, pid_begin=20_000_000, threads=1)
    dt1 = time.perf_counter() - t
    seg1 = r1["counters"]["segments"]
    return {"value": seg / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n2} histories of {spec['name']} (pids 1e7..), {seg} segments, {dt:.1f} s",
            "value_1core": seg1 / dt1,
            "sample_1core": f"{n1} histories (pids 2e7..), {seg1} segments, {dt1:.1f} s, 1 thread",
            "cpu_model": _cpu_model(),
            "falg_flops_per_segment": om.falg(r)}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(a, spec, rank, world):
    """--impl reference: the oracle (CPU) timed on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle
    om = oracle.OracleModel.from_spec(spec)
    cores = len(os.sched_getaffinity(0))
    probe = om.run(1000, seed=1, threads=cores)
    n = 2000
    t = time.perf_counter()
    om.run(n, seed=1, threads=cores)
    per = (time.perf_counter() - t) / n
    step_s = min(8.0, a.cpu_seconds)
    n_step = int(max(1000, min(2_000_000, step_s / max(per, 1e-9))))   # ~8 s per step
    for w in range(a.warmup):
        om.run(min(n_step, 20000), seed=100 + w, threads=cores)
    segs, tt = 0, 0.0
    for s in range(a.steps):
        t = time.perf_counter()
        r = om.run(n_step, seed=1000 + s, pid_begin=s * n_step, threads=cores)
        tt += time.perf_counter() - t
        segs += r["counters"]["segments"]
    v = segs / tt
    line = {"metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": 1e3 * tt / a.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": spec["name"], "histories_per_step": n_step, "tracker": "oracle (CPU)"},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{a.steps} steps x {n_step} histories of {spec['name']}"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    del probe
    print(json.dumps(line), flush=True)


def _free_port() -> int:
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def _self_launch(a):
    """`bench.py --gpus N` outside torchrun: re-exec as N ranks (one process per GPU) under
    torch.distributed.run on 127.0.0.1, the launch the driver uses for N > 1."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print(f"bench.py: launching {a.gpus} ranks: {' '.join(cmd)}", file=sys.stderr, flush=True)
    os.execv(sys.executable, cmd)


def main():
    a = _args()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        _self_launch(a)
    rank, world, local = _dist_env()
    if world != a.gpus:
        raise SystemExit(f"bench.py: --gpus {a.gpus} but WORLD_SIZE={world}; launch one rank per GPU")
    import workloads
    spec, n_cfg = workloads.config(a.config)
    if a.impl == "reference":
        run_reference(a, spec, rank, world)
        return

    import torch
    import paper_2406_13849_b200 as nt
    if not torch.cuda.is_available() or torch.cuda.device_count() <= local:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, "
                         f"{torch.cuda.device_count()} CUDA device(s) visible")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        if rank == 0:
            print(f"bench.py: {world} ranks, NCCL {'.'.join(map(str, torch.cuda.nccl.version()))}",
                  file=sys.stderr, flush=True)
    n = int(a.particles) if a.particles else n_cfg
    mesh_shape = None
    if a.mesh:
        mesh_shape = [int(v) for v in a.mesh.lower().split("x")]
        spec["mesh"] = {"lo": spec["source"]["lo"], "hi": spec["source"]["hi"], "shape": mesh_shape}
    model = nt.Model.from_spec(spec, device=local, pseudo_array=a.pseudo_array)
    mbuf = (torch.zeros(model.info["mesh_bins"], dtype=torch.float64, device="cuda")
            if mesh_shape else None)
    stream = torch.cuda.current_stream()
    out = torch.zeros(model.out_len, dtype=torch.float64, device="cuda")
    # L2 flush between timed steps: READ a 256 MB buffer (> 126 MB L2).  Reading leaves clean
    # lines, so no write-back of flush data is charged to the next tracking launch.
    flush = torch.ones(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    seed0 = workloads.SEED
    if a.tracker == "rect" and a.scheduler not in ("block", "history"):
        raise SystemExit("bench.py: the rect tracker runs on the ring queues (block) or history-based")
    kw = dict(tracker=a.tracker, block_dim=a.block_dim, blocks_per_sm=a.blocks_per_sm, scheduler=a.scheduler)

    outs = [torch.zeros(model.out_len, dtype=torch.float64, device="cuda") for _ in range(a.steps)]

    def step(s, o):
        o.zero_()
        if mbuf is not None:
            mbuf.zero_()
        model.track(n, seed=seed0 + s, pid_begin=rank * n, out=o, stream=stream, mesh=mbuf, **kw)
        if dist is not None:
            dist.all_reduce(o)      # the one collective: packed [len | exits | counters]

    for w in range(a.warmup):
        step(10_000 + w, out)
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    clocks = ClockSampler(local).start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(a.steps)]
    launches = 0
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    for s in range(a.steps):
        flush.max()                                 # evict L2 between timed steps (untimed)
        ev[s][0].record(stream)
        step(s, outs[s])
        ev[s][1].record(stream)
        launches += model.last_launch_count()
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    ck = clocks.stop()
    step_s = [e0.elapsed_time(e1) / 1e3 for e0, e1 in ev]
    t_rank = sum(step_s)
    t_max = t_rank
    if dist is not None:
        tt = torch.tensor([t_rank] + step_s, dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt[0])
        step_s = [float(x) for x in tt[1:]]          # per step: max over ranks
    per_step = [model.unpack(o) for o in outs]
    res = per_step[-1]
    segs = sum(p["counters"]["segments"] for p in per_step)      # all ranks (post all-reduce)
    particles = n * world * a.steps
    value = segs / t_max

    # kernel-only time on rank 0's stream is the same region (one launch per step), so the
    # kernel's average launch duration is t_rank / steps (all-reduce excluded only at N = 1)
    falg_doc = _load_json("falg.json") or {}
    falg = falg_doc.get(spec["name"])
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(spec, seed0, a.cpu_seconds)
        falg = cpu.pop("falg_flops_per_segment")
    peak = fp64_peak_tflops(ck["sm_max_mhz"])
    kernel_s = t_rank / a.steps
    achieved = (falg or 0.0) * (segs / (world * a.steps)) / kernel_s / 1e12 if falg else None
    traffic_doc = _load_json("traffic.json") or {}
    traffic = traffic_doc.get(_traffic_key(spec["name"], a, mesh_shape))
    hbm_peak = (_measured_peaks() or {}).get("hbm_gbs")
    hbm = None
    if traffic is not None and hbm_peak:
        gbs = traffic / kernel_s / 1e9
        hbm = {"bytes_per_launch": traffic, "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
               "frac": gbs / hbm_peak, "source": "ncu dram__bytes_read.sum + dram__bytes_write.sum of one "
               "launch (profiles/traffic.json) / this run's kernel time; peak MEASURED_PEAKS.json hbm_gbs"}
    frac = (achieved / peak) if achieved else None
    roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": frac,
            "traffic": traffic,
            "peak_source": "derived: 148 SM x 64 FP64 FMA/clk x 2 x sm_max_mhz (DESIGN.md)",
            "falg_flops_per_segment": falg, "kernel_ms_per_launch": 1e3 * kernel_s,
            "hbm": hbm,
            "binding": ("hbm" if hbm and frac is not None and hbm["frac"] > frac else "alu (fp64)")}

    # end to end right after the device-timed steps, under the same clocks (sampled here too)
    e2e = None
    ck_e2e = ClockSampler(local).start() if not a.no_e2e else None
    if not a.no_e2e and mbuf is not None:
        # mesh runs: the public Python call + D2H of the packed tallies and the mesh (pinned host)
        hout = torch.empty(model.out_len, dtype=torch.float64).pin_memory()
        hmesh = torch.empty(mbuf.numel(), dtype=torch.float64).pin_memory()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        esegs = 0
        t0 = time.perf_counter()
        e0.record(stream)
        for s in range(a.steps):
            out.zero_()
            mbuf.zero_()
            model.track(n, seed=seed0 + 500 + s, pid_begin=rank * n, out=out, stream=stream, mesh=mbuf, **kw)
            hout.copy_(out, non_blocking=True)
            hmesh.copy_(mbuf, non_blocking=True)
            torch.cuda.synchronize()
            esegs += int(hout[2 * model.n_mc + 1])
        e1.record(stream)
        torch.cuda.synchronize()
        te = max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0)
        e2e = {"value": esegs / te, "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(model.out_len * 8 + mbuf.numel() * 8),
               "api": "Model.track with a mesh buffer + D2H of tallies and mesh into pinned host memory"}
    elif not a.no_e2e:
        hout = None
        import numpy as np
        hout = np.zeros(model.out_len)
        for w in range(max(a.warmup, 1)):          # the same W full-size warm-up steps as the device timing
            model.track_host(n, seed=seed0 + 400 + w, pid_begin=rank * n, out=hout, stream=stream, **kw)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        esegs = 0
        if dist is not None:
            dist.barrier()
        t0 = time.perf_counter()
        e0.record(stream)
        step_ms, step_dev = [], []
        for s in range(a.steps):
            ts = time.perf_counter()
            d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            d0.record(stream)
            model.track_host(n, seed=seed0 + 500 + s, pid_begin=rank * n, out=hout, stream=stream, **kw)
            d1.record(stream)
            step_ms.append(1e3 * (time.perf_counter() - ts))
            step_dev.append((d0, d1))
            esegs += int(hout[2 * model.n_mc + 1])
        e1.record(stream)
        torch.cuda.synchronize()
        te = max(e0.elapsed_time(e1) / 1e3, time.perf_counter() - t0)
        if dist is not None:
            tt = torch.tensor([te, float(esegs)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tt[:1], op=dist.ReduceOp.MAX)
            dist.all_reduce(tt[1:], op=dist.ReduceOp.SUM)
            te, esegs = float(tt[0]), int(tt[1])
        e2e = {"value": esegs / te, "unit": UNIT, "h2d_bytes_per_step": 0,
               "d2h_bytes_per_step": int(model.out_len * 8),
               "api": "nt_track_host (host output buffer; births generated on device from seed/pid)",
               "note": "the method's per-step inputs are (seed, pid range): histories are born on the "
                       "device from Philox(seed, pid) (SURVEY O17/O18), so there are no input bytes to "
                       "copy; the D2H of the packed tallies is inside the timed region",
               "step_ms": [round(x, 1) for x in step_ms],
               "step_device_ms": [round(d0.elapsed_time(d1), 1) for d0, d1 in step_dev]}
    if ck_e2e is not None:
        ce = ck_e2e.stop()
        if e2e is not None:
            e2e["clocks"] = ce

    # the metric's second half: generic tree tracker vs the rect-specialised tracker, same histories
    ratio = None
    if not a.no_ratio and a.tracker == "generic" and model.info["rect_specialisable"]:
        def timed(kk):
            o2 = torch.zeros_like(out)
            model.track(n, seed=seed0 + 20_000, pid_begin=rank * n, out=o2, stream=stream, mesh=mbuf, **kk)
            torch.cuda.synchronize()
            tt, ss = 0.0, 0
            for s in range(a.steps):
                o2.zero_()
                flush.max()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                model.track(n, seed=seed0 + s, pid_begin=rank * n, out=o2, stream=stream, mesh=mbuf, **kk)
                e1.record(stream)
                torch.cuda.synchronize()
                tt += e0.elapsed_time(e1) / 1e3
                ss += model.unpack(o2)["counters"]["segments"]
            return ss / tt, ss
        rates, segs_seen = {}, set()
        for trk in ("generic", "rect"):
            for sch in ("block", "history"):
                r_, s_ = timed(dict(kw, tracker=trk, scheduler=sch))
                rates[f"{trk}_{sch}"] = r_
                segs_seen.add(s_)
        best_g = max(rates["generic_block"], rates["generic_history"])
        best_r = max(rates["rect_block"], rates["rect_history"])
        ratio = {"generic_over_rect": best_g / best_r,
                 "generic_ring_over_rect_ring": rates["generic_block"] / rates["rect_block"],
                 "generic_history_over_rect_history": rates["generic_history"] / rates["rect_history"],
                 "segments_per_s": rates, "segments_equal": len(segs_seen) == 1,
                 "note": "this rank, identical seeds/pids, no all-reduce, L2 flushed between steps; rect = the "
                         "Alg. 9-10 rect-specialised tracker; 'block' = the ring event-queue scheduler, "
                         "'history' = one history per thread; generic_over_rect = best scheduler of each "
                         "(north-star target >= 0.85); the same-scheduler ratios compare the trackers alone"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": 1e3 * t_max / a.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (histories born from Philox(seed, pid) on the device)",
                "config": {"workload": spec["name"], "histories_per_gpu_per_step": n,
                           "tracker": a.tracker, "pseudo_array": bool(a.pseudo_array),
                           "scheduler": kw["scheduler"],
                           "parallelism": f"pid-sharded x{world}, one fp64 all-reduce per step",
                           "l2": "256 MB buffer read between timed steps (L2 flushed)",
                           "mesh_tally": mesh_shape},
                "particles_per_s": particles / t_max,
                "step_ms": [round(1e3 * x, 3) for x in step_s],
                "ms_per_step_median": 1e3 * _median(step_s),
                "cv": _cv(step_s),
                "segments_per_s_median_step": segs / a.steps / _median(step_s),
                "segments_per_history": segs / particles,
                "counters_last_step": res["counters"],
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "rect_ratio": ratio,
                "gpu_launches": launches, "clocks": ck}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def _median(x):
    y = sorted(x)
    k = len(y)
    return y[k // 2] if k % 2 else 0.5 * (y[k // 2 - 1] + y[k // 2])


def _cv(x):
    if len(x) < 2:
        return None
    m = sum(x) / len(x)
    var = sum((v - m) ** 2 for v in x) / (len(x) - 1)
    return var ** 0.5 / m


if __name__ == "__main__":
    main()
