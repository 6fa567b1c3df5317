"""Multi-rank DEVICE path: two ranks on cuda:0 (the GPU box has one GPU; NCCL
refuses two ranks on one device, so the process group is gloo, which stages the tensors through
the host).  Unlike tests/test_distributed_cpu.py, nothing is injected: `track_distributed` and
`power_iteration_distributed` call nt_track / nt_bank_compact / nt_source_from_sites, and the
combined result is compared with the oracle at world size 1."""
import os
import socket

import numpy as np
import pytest

import workloads

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _track_worker(rank, world, port, cfg, n, seed, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2406_13849_b200 as nt
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    spec, _ = workloads.config(cfg)
    m = nt.Model.from_spec(spec, device=0)
    stream = torch.cuda.Stream()                 # a non-default stream: ordering must follow it
    with torch.cuda.stream(stream):
        out = nt.track_distributed(m, n, seed, pid_begin=0)
    stream.synchronize()
    assert out.is_cuda
    np.save(os.path.join(outdir, f"out_{rank}.npy"), out.cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg,n", [("c2", 3001), ("c3", 2001), ("c4", 1501)])
def test_two_rank_device_track_distributed(tmp_path, oracle_mod, cfg, n):
    port = _free_port()
    mp.spawn(_track_worker, args=(2, port, cfg, n, 5, str(tmp_path)), nprocs=2, join=True)
    o0, o1 = np.load(tmp_path / "out_0.npy"), np.load(tmp_path / "out_1.npy")
    assert np.array_equal(o0, o1)
    spec, _ = workloads.config(cfg)
    om = oracle_mod.OracleModel.from_spec(spec)
    full = om.run(n, seed=5)
    got = om.unpack(o0)
    assert got["counters"] == full["counters"]
    assert got["counters"]["particles"] == n
    assert np.array_equal(got["exits"], full["exits"])
    assert np.allclose(got["len"], full["len"], rtol=1e-12, atol=0)


def _pi_worker(rank, world, port, n, cycles, outdir):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2406_13849_b200 as nt
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    m = nt.Model.from_spec(workloads.with_fission(workloads.c2_assembly(), {"uo2": 0.30}), device=0)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        ks = nt.power_iteration_distributed(m, n, cycles, seed=21)
    stream.synchronize()
    np.save(os.path.join(outdir, f"ks_{rank}.npy"), np.array(ks))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_device_power_iteration(tmp_path, oracle_mod):
    """F1 across ranks through the device calls: 2 ranks x n = one process with 2n histories."""
    port = _free_port()
    n, cycles = 1500, 3
    mp.spawn(_pi_worker, args=(2, port, n, cycles, str(tmp_path)), nprocs=2, join=True)
    k0, k1 = np.load(tmp_path / "ks_0.npy"), np.load(tmp_path / "ks_1.npy")
    assert np.array_equal(k0, k1)
    om = oracle_mod.OracleModel.from_spec(workloads.with_fission(workloads.c2_assembly(), {"uo2": 0.30}))
    ref = om.power_iteration(2 * n, cycles, seed=21)
    assert np.array_equal(k0, np.array(ref))
