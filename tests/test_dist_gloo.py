"""N>1 host path on CPU with gloo (world_size 2): each rank owns a disjoint
shard of the synthetic workload (weak scaling, no data-path collective) and
the timing reduction is the max over ranks."""

from __future__ import annotations

import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    segs = bench.make_workload(8, rank)
    t = bench.max_over_ranks(float(10 + rank), world)
    bench.barrier(world)
    q.put((rank, [u for u, _ in segs], t))
    dist.destroy_process_group()


def test_weak_scaling_shards_and_max_over_ranks():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    ids0, ids1 = set(out[0][1]), set(out[1][1])
    assert len(ids0) == 8 and len(ids1) == 8 and not ids0 & ids1
    assert out[0][2] == out[1][2] == 11.0
