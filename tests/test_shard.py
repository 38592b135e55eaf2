"""Multi-rank host logic on CPU (gloo, world_size 2): pair shards are disjoint
and cover the batch, the per-rank generator inputs are exactly the single-rank
batch split by pair, the max-over-ranks timing reduction and the result
gather behave. (The compute path itself needs no collective.)"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2205_03133_b200.shard import strong_shard, weak_shard


def test_shard_math():
    assert [weak_shard(4, r, 3) for r in range(3)][2].start == 8
    parts = [strong_shard(10, r, 4) for r in range(4)]
    assert sum(p.count for p in parts) == 10
    assert [p.start for p in parts] == [0, 2, 5, 7]
    with pytest.raises(ValueError):
        weak_shard(4, 3, 3)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    import paper_2205_03133_b200 as P
    from paper_2205_03133_b200.shard import gather_to_rank0, max_over_ranks, weak_shard

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sh = weak_shard(2, rank, world)
    left, right = P.synth_batch(0, sh.count, seed0=sh.start, threads=1, width=64, height=48)
    t = max_over_ranks(1.0 + rank)
    gathered = gather_to_rank0(left)
    if rank == 0:
        q.put(("max", t))
        q.put(("left", gathered))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo(built):
    import paper_2205_03133_b200 as P

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got["max"] == 2.0
    single, _ = P.synth_batch(0, 4, seed0=0, threads=1, width=64, height=48)
    assert np.array_equal(got["left"], single)
