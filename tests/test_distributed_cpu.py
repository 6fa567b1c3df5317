"""Multi-rank path on CPU (gloo, world size 2): contiguous pid sharding + one all-reduce of the
packed [len | exits | counters] buffer.  The per-rank tracker here is the oracle
(no GPU in this container); on a GPU box the same `track_distributed` calls nt_track."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, cfg, n, seed, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_2406_13849_b200 as nt
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    spec, _ = workloads.config(cfg)
    om = oracle.OracleModel.from_spec(spec)
    seen = []

    def tracker(nn, pid0):
        seen.append((pid0, nn))
        return torch.from_numpy(om.run(nn, seed=seed, pid_begin=pid0, threads=1)["out"].copy())

    out = nt.track_distributed(None, n, seed, pid_begin=0, tracker_fn=tracker)
    np.save(os.path.join(outdir, f"out_{rank}.npy"), out.numpy())
    np.save(os.path.join(outdir, f"shard_{rank}.npy"), np.array(seen[0]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n", [("c2", 301), ("c3", 257)])
def test_two_rank_sharding_allreduce(tmp_path, oracle_mod, cfg, n):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, cfg, n, 5, str(tmp_path)), nprocs=2, join=True)
    o0 = np.load(tmp_path / "out_0.npy")
    o1 = np.load(tmp_path / "out_1.npy")
    assert np.array_equal(o0, o1)                       # every rank holds the combined tally
    s0, s1 = np.load(tmp_path / "shard_0.npy"), np.load(tmp_path / "shard_1.npy")
    assert tuple(s0) == (0, n // 2) and tuple(s1) == (n // 2, n - n // 2)   # contiguous shards
    spec, _ = workloads.config(cfg)
    om = oracle_mod.OracleModel.from_spec(spec)
    full = om.run(n, seed=5, threads=1)
    got = om.unpack(o0)
    assert got["counters"] == full["counters"]          # exact for any world size
    assert np.array_equal(got["exits"], full["exits"])
    assert np.allclose(got["len"], full["len"], rtol=1e-13, atol=0)


def test_shard_function():
    import paper_2406_13849_b200 as nt
    for N in (0, 1, 7, 100, 10**8 + 3):
        for G in (1, 2, 3, 8):
            shards = [nt.shard(N, g, G) for g in range(G)]
            assert sum(k for _, k in shards) == N
            assert all(shards[g][0] + shards[g][1] == (shards[g + 1][0] if g + 1 < G else N) for g in range(G))


def _pi_worker(rank, world, port, n, cycles, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import oracle
    import paper_2406_13849_b200 as nt
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    om = oracle.OracleModel.from_spec(workloads.infinite_medium(1.0, 0.25, 0.55))

    def track(nn, pid0, states, cycle):
        res = om.run(nn, seed=21, pid_begin=pid0, bank=True, threads=1,
                     states=None if states is None else states.numpy())
        sites = om.bank_sites(res["bank"], res["bank_n"])
        return torch.from_numpy(sites.copy()), len(sites)

    def sample(sites, M, cycle, j0, nn):
        return torch.from_numpy(om.source_from_sites(sites.numpy(), 21, cycle, j0, nn).copy())

    ks = nt.power_iteration_distributed(None, n, cycles, seed=21, track_fn=track, sample_fn=sample)
    np.save(os.path.join(outdir, f"ks_{rank}.npy"), np.array(ks))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_power_iteration_allgather(tmp_path, oracle_mod):
    """Multi-rank power iteration (F1): the all-gathered fission bank makes 2 ranks x n histories
    reproduce one process tracking 2n histories, cycle by cycle (k exact)."""
    port = _free_port()
    n, cycles = 300, 3
    mp.spawn(_pi_worker, args=(2, port, n, cycles, str(tmp_path)), nprocs=2, join=True)
    k0, k1 = np.load(tmp_path / "ks_0.npy"), np.load(tmp_path / "ks_1.npy")
    assert np.array_equal(k0, k1)
    om = oracle_mod.OracleModel.from_spec(workloads.infinite_medium(1.0, 0.25, 0.55))
    ref = om.power_iteration(2 * n, cycles, seed=21)
    assert np.array_equal(k0, np.array(ref))


def test_bench_gpus_flag_launches_ranks():
    """`bench.py --gpus 2` outside torchrun re-launches itself as 2 ranks (reference arm: runs on
    CPU here); rank 0 alone prints the one JSON line, with n_gpus = 2."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    p = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "0", "--config", "c1", "--cpu-seconds", "0.5"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=root)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    assert "launching 2 ranks" in p.stderr
