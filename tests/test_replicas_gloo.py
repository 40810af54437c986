"""Multi-process (world_size 2, gloo on CPU) checks of the replica bookkeeping
used by `bench.py --gpus N`: request batches shard round-robin, and the
whole-job value is the sum of tokens over the max of per-rank seconds."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2604_26334_b200.runtime.replicas import aggregate, shard_batches


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard_batches(list(range(7)), rank, world)
    # rank r "decodes" 32 tokens per batch it owns, taking (r + 1) seconds
    out = aggregate(tokens=32 * len(mine), seconds=float(rank + 1))
    dist.barrier()
    q.put((rank, mine, out))
    dist.destroy_process_group()


def test_two_replicas_aggregate_over_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    results = dict()
    for _ in range(world):
        rank, mine, out = q.get(timeout=120)
        results[rank] = (mine, out)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert results[0][0] == [0, 2, 4, 6] and results[1][0] == [1, 3, 5]
    for rank in range(world):
        out = results[rank][1]
        assert out["world"] == 2
        assert out["tokens"] == 32 * 7
        assert out["seconds_max"] == 2.0
        assert out["value"] == pytest.approx(32 * 7 / 2.0)


def test_single_process_aggregate_is_local():
    out = aggregate(tokens=10, seconds=2.0)
    assert out == {"tokens": 10, "seconds_max": 2.0, "value": 5.0, "world": 1}


def _shared_name_worker(rank, world, port, q):
    import os

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2604_26334_b200.runtime.replicas import shared_weights_name
    q.put((rank, shared_weights_name("tiny-llama")))
    dist.destroy_process_group()


def test_shared_weights_name_agreed_across_ranks():
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_shared_name_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(60)
    names = dict(q.get(timeout=10) for _ in range(2))
    assert names[0] == names[1] and names[0].startswith("pshard_tiny-llama_0_")
