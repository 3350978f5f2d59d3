"""Multi-process (world_size 2, gloo, CPU) checks of the batch-sharded path:
shards partition the batch, per-shard transforms equal the whole-batch
transform, MAX-over-ranks timing reduce.  The GPU leg runs the same code with
the nccl backend (bench.py under torchrun)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2104_11471_b200.shard import gather_shards, max_over_ranks, my_shard, shard_range


@pytest.mark.parametrize("batch,world", [(16384, 8), (64, 8), (7, 2), (1, 4), (1024, 3)])
def test_shards_partition_batch(batch, world):
    seen = []
    for r in range(world):
        s, e = shard_range(batch, r, world)
        seen.extend(range(s, e))
        assert e - s in (batch // world, batch // world + 1)
    assert seen == list(range(batch))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, batch, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import restate as R

        x = R.random_pairs([5, n], batch, n)  # every rank can regenerate the global input
        sh = my_shard(batch)
        y_local = torch.from_numpy(R.fft_half(x[sh.start: sh.stop]).view(np.uint16).astype(np.int32))
        y = gather_shards(y_local, batch)
        t = max_over_ranks(float(rank + 1))
        if rank == 0:
            full = R.fft_half(x).view(np.uint16).astype(np.int32)
            q.put((bool(np.array_equal(y.numpy(), full)), t))
    finally:
        dist.destroy_process_group()


def test_sharded_transform_equals_whole_batch_gloo():
    world, n, batch = 2, 256, 7
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, batch, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    ok, tmax = q.get(timeout=10)
    assert ok
    assert tmax == float(world)
    assert all(p.exitcode == 0 for p in procs)
