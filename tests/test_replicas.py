"""Multi-process (world_size 2, gloo, CPU) check of bench.py's N > 1 host logic: the path does not
shard (north_star: one GPU, no collectives), so every rank runs an independent replica and the only
collective is the max over ranks of the device-timed region."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    sys.path.insert(0, ROOT)
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms_local = [3.0, 5.0][rank]                       # rank 1 is the slower replica
    ms = bench.max_over_ranks(ms_local, dist, torch.device("cpu"))
    val = bench.aggregate_value(1000, 10, ms, world)
    out[rank] = (ms, val)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_replicas_gloo():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        ms, val = out[r]
        assert ms == 5.0                                  # max over ranks
        assert val == pytest.approx(world * 1000 * 10 / 5e-3)


def test_single_rank_is_identity():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.max_over_ranks(2.5, None, None) == 2.5
    assert bench.aggregate_value(10, 4, 2.0, 1) == pytest.approx(10 * 4 / 2e-3)
