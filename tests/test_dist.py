"""Replica (N > 1) aggregation of bench.py on CPU with gloo, world_size 2."""

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

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # rank 1 is slower: the job time must be the max over ranks
    times = [100.0, 110.0] if rank == 0 else [150.0, 160.0]
    v, total = bench.aggregate(times, world, 49200, reduce_max)
    out[rank] = (v, total)
    dist.barrier()
    dist.destroy_process_group()


def test_replicas_max_over_ranks():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    assert out[0] == out[1]
    v, total = out[0]
    assert total == pytest.approx(310.0)
    assert v == pytest.approx(2 * 2 * 49200 / 0.310)
