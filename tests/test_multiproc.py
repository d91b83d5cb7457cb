"""N > 1 bench path on the CPU: two gloo ranks run independent oracle replicas
(the hot path does not shard -- DESIGN.md section 7), and the timing
aggregation bench.py uses (max over ranks, whole-job rate) is exercised over a
real process group."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from oracle import oracle as O
    from tests.golden import fixtures
    z, h = fixtures.load("c1s")
    # each rank: an independent replica of the same seeded V-cycle
    u = z["g/u_rand"].copy()
    O.vcycle(h, z["g/b"], u)
    rel = float(np.linalg.norm(u - z["g/vcycle1"]) / np.linalg.norm(z["g/vcycle1"]))
    elapsed = 0.5 + rank  # rank-dependent synthetic elapsed time
    mx = bench.max_over_ranks(elapsed, device="cpu")
    rate = bench.whole_job_rate(10, mx, world)
    out[rank] = (rel, mx, rate)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_and_timing_aggregation():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for rank in range(world):
        rel, mx, rate = out[rank]
        assert rel <= 1e-12
        assert mx == 1.5                   # max over ranks
        assert rate == pytest.approx(world * 10 / 1.5)
