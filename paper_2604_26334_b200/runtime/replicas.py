"""Batched mode across GPUs: independent data-parallel replicas.

One process per GPU; each replica owns whole request batches, its own capped
arena, its own plan (identical inputs give an identical plan) and its own host
link. Nothing is reduced across GPUs on the data path — no NCCL collective
touches activations or weights. The only cross-rank traffic is bookkeeping:
a barrier around the timed region and a max / sum of per-rank scalars.
"""

from __future__ import annotations

import os


def rank_world() -> tuple[int, int, int]:
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def shard_batches(batches: list, rank: int, world: int) -> list:
    """Request batches round-robin over replicas (batch i -> rank i % world)."""
    return [b for i, b in enumerate(batches) if i % world == rank]


def aggregate(tokens: int, seconds: float, device: str = "cpu") -> dict:
    """Whole-job throughput of independent replicas.

    value = (sum of tokens over ranks) / (max of device seconds over ranks):
    the job finishes when its slowest replica does. Works on any initialised
    torch.distributed backend (gloo on CPU tensors, NCCL on CUDA tensors);
    without one it returns the local numbers."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return {"tokens": tokens, "seconds_max": seconds, "value": tokens / seconds, "world": 1}
    t = torch.tensor([float(tokens)], dtype=torch.float64, device=device)
    s = torch.tensor([float(seconds)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    dist.all_reduce(s, op=dist.ReduceOp.MAX)
    total, slowest = float(t.item()), float(s.item())
    return {"tokens": total, "seconds_max": slowest, "value": total / slowest,
            "world": dist.get_world_size()}


def shared_weights_name(model: str, seed: int = 0) -> str | None:
    """A /dev/shm segment name every replica of this job agrees on (rank 0 draws a
    random token and broadcasts it), or None outside torch.distributed. Replicas on
    one node then hold one host copy of the weights (model.SharedHostBlob)."""
    import secrets

    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return None
    box = [secrets.token_hex(6) if dist.get_rank() == 0 else None]
    dist.broadcast_object_list(box, src=0)
    return f"pshard_{model}_{seed}_{box[0]}"
