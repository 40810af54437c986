"""Residency-migration cost model and migration-aware tier choice.

SURVEY.md §8f row 3. The reference charges a tier switch nothing: its
SetupForSched is free (`SPEC.md:430`, `pkg/src/shardplan/simulator.py:239-314`
never prices a residency change). On a real GPU a switch moves bytes — KV
caches that leave VRAM go home over D2H, newly pinned weights and KV caches
come in over H2D — and the executor measures exactly those bytes
(`Executor.set_tier`). This module predicts them from the plans alone, with
the executor's own policy:

1. every VRAM-pinned KV cache of the old tier is written home: its live pages
   (`kv_pages * page_bytes` each; the paged cache, executor.KvPagePool);
2. the new tier's pinned set is carved bottom-up in pin order
   (priority, layer, id), 256-byte aligned, followed by the executor's spare
   pins (`Executor.pins_for`); a weight shard whose offset is unchanged stays,
   one resident in both tiers at different offsets is relocated inside VRAM
   (device-to-device, `plan_relocation`: no link bytes), every other pinned
   weight is uploaded whole;
3. every VRAM-pinned KV cache of the new tier is uploaded (same pages).

`seconds()` prices the bytes on the machine's link rates (the executor runs
the copies back to back on one stream). `pick_tier()` is the reference's
`pick_tier` rule (`pkg/src/shardplan/planner.py:451-460`: argmin over ascending
tiers of ceil(n / t) * time[t], strict <) plus the migration seconds of
switching from the current tier — an extension the engine applies only when
asked (`Engine(..., migration_aware=True)`), so the default loop stays the
reference's.
"""

from __future__ import annotations

import os

from ..planning.graph import ShardKind, build_shards
from ..planning.hardware import MachineSpec
from ..planning.placement import TIERS, Residency, SchedulePlan

ALIGN = 256


def _up(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


def plan_relocation(old: dict, new: dict, max_pieces: int = 64) -> tuple[list, list]:
    """Move weight shards between two layouts of ONE arena without the host link.

    old / new: shard id -> (offset, bytes). Returns (d2d, h2d): d2d is an ordered
    list of (sid, src, dst, bytes) device-to-device copies that never overwrite a
    source still to be read — a shard moves only once its destination overlaps no
    other pending shard's source; a shard overlapping its own source moves in
    pieces no longer than the shift (ascending when it moves down, descending when
    up; more than `max_pieces` pieces and it is uploaded instead); a dependency
    cycle is broken by uploading its smallest shard from the host — and h2d the shard ids
    to upload afterwards (not resident before, or cycle breakers), in `new` order.
    Shards at an unchanged offset appear in neither. Pure and deterministic: the
    executor runs it and the migration model prices it."""
    def overlaps(a0, n0, a1, n1):
        return a0 < a1 + n1 and a1 < a0 + n0

    def pieces(sid):
        (src, n), dst = old[sid], new[sid][0]
        if not overlaps(src, n, dst, n):
            return [(sid, src, dst, n)]
        c = abs(dst - src)
        out = [(sid, src + o, dst + o, min(c, n - o)) for o in range(0, n, c)]
        return out if dst < src else out[::-1]

    h2d = [sid for sid in new if sid not in old]
    if os.environ.get("PS_RELOCATE", "1") == "0":   # A/B switch: upload every moved shard
        return [], h2d + [sid for sid in new if sid in old and old[sid][0] != new[sid][0]]
    pending = sorted((sid for sid in new if sid in old and old[sid][0] != new[sid][0]),
                     key=lambda sid: (new[sid][0], sid))
    fallback = set()
    for sid in list(pending):
        (src, n), dst = old[sid], new[sid][0]
        if overlaps(src, n, dst, n) and -(-n // abs(dst - src)) > max_pieces:
            pending.remove(sid)
            fallback.add(sid)
    d2d = []
    while pending:
        for sid in pending:
            dst, n = new[sid]
            if not any(o != sid and overlaps(dst, n, old[o][0], old[o][1]) for o in pending):
                d2d += pieces(sid)
                pending.remove(sid)
                break
        else:   # every pending move would clobber another's source: upload the smallest
            victim = min(pending, key=lambda sid: (new[sid][1], new[sid][0], sid))
            pending.remove(victim)
            fallback.add(victim)
    h2d += [sid for sid in new if sid in fallback]
    return d2d, h2d


class MigrationModel:
    def __init__(self, spec, layout, plans: dict, context_len: int, batch: int, pins_fn=None):
        self.spec, self.plans = spec, plans
        # tier -> shard ids in carve order; the executor's pins_for adds its spare pins
        self.pins_fn = pins_fn
        self.phys_fn = None
        self.shards = build_shards(spec, context_len, batch)
        self.batch = batch
        from .executor import KV_PAGE_ROWS
        self.row_bytes = 2 * spec.n_kv_heads * spec.head_dim * 2
        self.page_bytes = KV_PAGE_ROWS * self.row_bytes
        self.kv_layer_bytes = batch * -(-context_len // KV_PAGE_ROWS) * self.page_bytes
        self.blob_bytes = {sid: b.nbytes for sid, b in layout.blobs.items()}

    def _phys(self, shard) -> int:
        if shard.kind is ShardKind.KV_CACHE:
            return self.kv_layer_bytes
        if self.phys_fn is not None:     # the executor's resident size (coded shards: smaller)
            return self.phys_fn(shard.id)
        return self.blob_bytes[shard.id]

    def pinned_offsets(self, tier: int) -> dict:
        """shard id -> arena offset of every VRAM-resident shard at `tier` (executor
        carve order: the plan's pins in pin order, then any spare pins)."""
        if self.pins_fn is not None:
            sids = self.pins_fn(tier)
        else:
            plan = self.plans[tier]
            sids = [p.shard_id for p in sorted(
                (p for p in plan.placements if p.residency is Residency.VRAM_PINNED),
                key=lambda p: (self.shards[p.shard_id].priority, self.shards[p.shard_id].layer_index,
                               p.shard_id))]
        out, off = {}, 0
        for sid in sids:
            out[sid] = off
            off += _up(self._phys(self.shards[sid]))
        return out

    def bytes(self, from_tier: int | None, to_tier: int, kv_pages: int) -> tuple[int, int]:
        """(h2d, d2h) bytes of switching from `from_tier` (None: nothing resident)
        to `to_tier` with `kv_pages` live KV pages per layer."""
        if from_tier == to_tier:
            return 0, 0
        return self.moves(from_tier, to_tier, kv_pages)[:2]

    def moves(self, from_tier: int | None, to_tier: int, kv_pages: int) -> tuple[int, int, int]:
        """(h2d, d2h, d2d) bytes of the switch; d2d never crosses the host link."""
        if from_tier == to_tier:
            return 0, 0, 0
        rows_bytes = kv_pages * self.page_bytes
        old = self.pinned_offsets(from_tier) if from_tier is not None else {}
        new = self.pinned_offsets(to_tier)
        kv = lambda sid: self.shards[sid].kind is ShardKind.KV_CACHE  # noqa: E731
        d2h = sum(rows_bytes for sid in old if kv(sid))
        h2d = sum(rows_bytes for sid in new if kv(sid))
        w_old = {sid: (off, self._phys(self.shards[sid])) for sid, off in old.items() if not kv(sid)}
        w_new = {sid: (off, self._phys(self.shards[sid])) for sid, off in new.items() if not kv(sid)}
        d2d, up = plan_relocation(w_old, w_new)
        h2d += sum(w_new[sid][1] for sid in up)
        return h2d, d2h, sum(op[3] for op in d2d)

    def seconds(self, from_tier, to_tier, kv_pages: int, machine: MachineSpec) -> float:
        h2d, d2h = self.bytes(from_tier, to_tier, kv_pages)
        return h2d / machine.pcie_h2d_bw + d2h / machine.pcie_d2h_bw

    def pick_tier(self, n_new: int, current: int | None, kv_pages: int, machine: MachineSpec) -> int:
        """Reference pick_tier over reachable tiers, plus the switch cost."""
        best, best_cost = None, None
        for tier in TIERS:
            plan = self.plans.get(tier)
            if plan is None:
                continue
            cost = -(-n_new // tier) * plan.estimated_time
            if current is not None and tier != current:
                cost = cost + self.seconds(current, tier, kv_pages, machine)
            if best_cost is None or cost < best_cost:
                best, best_cost = tier, cost
        return best
