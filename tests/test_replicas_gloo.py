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


def _engine_replica(rank, world, port, name, q):
    """One replica of `bench.py --gpus 2` on ONE GPU: gloo bookkeeping, node-shared
    host weights AND node-shared exponent-coded copy (one replica encodes)."""
    import sys
    sys.path.insert(0, os.getcwd())
    import numpy as np
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2604_26334_b200.planning import catalog
        from paper_2604_26334_b200.planning.graph import total_model_bytes
        from paper_2604_26334_b200.runtime.engine import Engine
        spec = catalog.builtin_model("tiny-llama")
        eng = Engine(spec, budget_bytes=0.3 * total_model_bytes(spec), context_len=160, batch=2,
                     shared_weights=name)
        prompts = [np.random.default_rng(70 + rank * 2 + i).integers(0, spec.vocab_size, 40).astype(np.int32)
                   for i in range(2)]
        res = eng.generate(prompts, gen_len=12)
        dist.barrier()
        coded = eng.weights.coded
        info = (eng.weights.shared is not None and eng.weights.shared.creator,
                coded is not None and coded.seg is not None, coded is not None and coded.seg is not None
                and coded.seg.creator)
        out = aggregate(tokens=2 * 11, seconds=res.decode_time_s)
        q.put((rank, [t.tolist() for t in res.tokens], info, out["world"]))
        dist.barrier()
        eng.close()
        dist.destroy_process_group()
    except BaseException as exc:   # report instead of leaving the parent waiting
        import traceback
        q.put((rank, "".join(traceback.format_exception(exc)), None, None))
        raise


@pytest.mark.gpu
def test_two_engine_replicas_match_single_runs():
    """`bench.py --gpus 2` run-readiness on a one-GPU box: two Engine replicas (gloo for
    the bookkeeping, no NCCL) share ONE host copy of the weights and ONE coded copy —
    exactly one replica creates each — and every replica's tokens equal the same
    requests run by a lone engine."""
    import secrets
    import numpy as np
    from paper_2604_26334_b200.planning import catalog
    from paper_2604_26334_b200.planning.graph import total_model_bytes
    from paper_2604_26334_b200.runtime.engine import Engine
    spec = catalog.builtin_model("tiny-llama")
    name = "pshard_rep_" + secrets.token_hex(4)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_engine_replica, args=(r, world, port, name, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(world):
        rank, toks, info, w = q.get(timeout=300)
        assert info is not None, toks
        got[rank] = (toks, info, w)
    for p in procs:
        p.join(60)
    assert sorted(got[r][1][0] for r in got) == [False, True]      # one creator of the weights
    assert all(got[r][1][1] for r in got)                           # both stream the shared coded copy
    assert sorted(got[r][1][2] for r in got) == [False, True]      # one encoder
    assert all(got[r][2] == world for r in got)
    for rank in range(world):
        eng = Engine(spec, budget_bytes=0.3 * total_model_bytes(spec), context_len=160, batch=2)
        prompts = [np.random.default_rng(70 + rank * 2 + i).integers(0, spec.vocab_size, 40).astype(np.int32)
                   for i in range(2)]
        want = eng.generate(prompts, gen_len=12)
        eng.close()
        assert got[rank][0] == [t.tolist() for t in want.tokens], rank
    assert not os.path.exists(f"/dev/shm/{name}") and not os.path.exists(f"/dev/shm/{name}_coded")
