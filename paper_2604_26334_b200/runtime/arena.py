"""Capped VRAM arena: the whole VRAM budget is ONE device allocation.

Row a24 of SURVEY.md §8: the plan splits the budget into a pinned region
and scratch (`pkg/src/shardplan/planner.py:159`); the reference checks VRAM
demand only in simulation (`pkg/src/shardplan/simulator.py:136-145`). Here
the budget is physical: `budget` bytes are allocated once, and every
device buffer of the executor — pinned shards, pinned KV caches, the
staging ring, activations, small fixed tables — is carved out of it.
Pinned shards grow bottom-up, transient regions (ring, activations) are
carved top-down; a request that does not fit raises `ArenaExhausted`
instead of silently allocating elsewhere.
"""

from __future__ import annotations

from ..planning.faults import ShardPlanError

ALIGN = 256


class ArenaExhausted(ShardPlanError):
    """A carve-out would exceed the VRAM budget."""


def _up(n: int, a: int = ALIGN) -> int:
    return (n + a - 1) // a * a


class VramArena:
    def __init__(self, budget_bytes: int, device: str = "cuda"):
        import torch
        self.capacity = int(budget_bytes) // ALIGN * ALIGN
        self._buf = torch.empty(self.capacity, dtype=torch.uint8, device=device)
        self.base = self._buf.data_ptr()
        self.low = 0                 # bottom-up cursor (persistent: pinned shards, KV)
        self.high = self.capacity    # top-down cursor (transient: ring, activations)
        self.low_marks: dict[str, tuple[int, int]] = {}
        self.high_marks: dict[str, tuple[int, int]] = {}

    # -- bottom-up (persistent) --------------------------------------------------
    def alloc_low(self, tag: str, nbytes: int) -> int:
        n = _up(nbytes)
        if self.low + n > self.high:
            raise ArenaExhausted(
                f"arena: '{tag}' needs {n} B, only {self.high - self.low} B free of "
                f"{self.capacity} B budget")
        off = self.low
        self.low += n
        self.low_marks[tag] = (off, n)
        return self.base + off

    def reset_low(self) -> None:
        self.low = 0
        self.low_marks.clear()

    # -- top-down (transient) ----------------------------------------------------
    def alloc_high(self, tag: str, nbytes: int) -> int:
        n = _up(nbytes)
        if self.high - n < self.low:
            raise ArenaExhausted(
                f"arena: '{tag}' needs {n} B, only {self.high - self.low} B free of "
                f"{self.capacity} B budget")
        self.high -= n
        self.high_marks[tag] = (self.high, n)
        return self.base + self.high

    def reset_high(self) -> None:
        self.high = self.capacity
        self.high_marks.clear()

    @property
    def free_bytes(self) -> int:
        return self.high - self.low

    @property
    def used_bytes(self) -> int:
        return self.low + (self.capacity - self.high)

    def tensor(self, ptr: int, nbytes: int):
        """uint8 torch view of a carved range (tests / debugging)."""
        off = ptr - self.base
        return self._buf[off:off + nbytes]
