"""N > 1 host logic on CPU: world-size-2 gloo process group, the bench's max-over-ranks timing and the
whole-job aggregation (replicas of independent factorizations, "scaling": "weak")."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    t = bench.max_over_ranks(100.0 + 50.0 * rank)  # rank 1 is the slow one
    v = bench.aggregate_value(1e12, 3, world, t)
    out[rank] = (t, v)
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_and_aggregate_gloo():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        t, v = out[r]
        assert t == 150.0  # max over ranks
        assert abs(v - 1e12 * 3 * 2 / 0.150 / 1e12) < 1e-9


def test_single_process_passthrough():
    import bench

    assert bench.max_over_ranks(12.5) == 12.5
    assert abs(bench.aggregate_value(2e12, 2, 1, 1000.0) - 4.0) < 1e-12
