"""N > 1 bench path on CPU (gloo, world_size 2): the path does not shard, every rank
runs a replica; the job time is the max over ranks and the value the whole-job rate."""
from __future__ import annotations

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


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench

    ms = 100.0 + 50.0 * rank  # rank 1 is the slow replica
    got = bench.max_over_ranks(ms, dist)
    q.put((rank, got, bench.job_value(1000, world, 4, got)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_max_over_ranks_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in procs)
    for p in procs:
        p.join(30)
    assert [r[1] for r in res] == [150.0, 150.0]
    # 2 ranks x 1000 vertices x 4 steps in 150 ms
    assert abs(res[0][2] - 2 * 1000 * 4 / 0.150 / 1e6) < 1e-12


def test_single_rank_passthrough():
    import bench

    assert bench.max_over_ranks(12.5, None) == 12.5
