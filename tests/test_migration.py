"""Residency-migration cost model (runtime/migration.py) on CPU: plan-only
predictions, the reference pick_tier rule when switches are free, and that a
switch with a large cost is avoided. The bytes are checked against the
executor's measured switches in test_engine_gpu.py."""

import pytest

from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.planning.costdb import synth_profile
from paper_2604_26334_b200.planning.graph import ShardKind, total_model_bytes
from paper_2604_26334_b200.planning.placement import TIERS, Residency, reachable_tiers
from paper_2604_26334_b200.runtime.migration import MigrationModel
from paper_2604_26334_b200.runtime.model import WeightLayout, arch_for


def _model(name, frac=None, budget=None, ctx=2304, batch=1):
    spec = catalog.builtin_model(name)
    m = catalog.builtin_machine("b200")
    budget = budget or frac * total_model_bytes(spec)
    plans = reachable_tiers(spec, m, synth_profile(m), budget, ctx, batch)
    return spec, m, plans, MigrationModel(spec, WeightLayout(spec, arch_for(spec)), plans, ctx, batch)


def test_fresh_executor_uploads_every_pinned_shard():
    spec, m, plans, mm = _model("llama3.1-8b", budget=4e9)
    for tier, plan in plans.items():
        h2d, d2h = mm.bytes(None, tier, 0)   # plan-only model (no executor spare pins)
        assert d2h == 0
        want = sum(mm._phys(mm.shards[p.shard_id]) for p in plan.placements
                   if p.residency is Residency.VRAM_PINNED and mm.shards[p.shard_id].kind is not ShardKind.KV_CACHE)
        assert h2d == want
        assert mm.bytes(tier, tier, 100) == (0, 0)


def test_l8_decode_prefill_switch_bytes():
    """Config 2: the decode tier pins 22 attention + 5 KV shards, tier 2048 pins 21
    attention: switching to prefill writes 5 KV caches home."""
    spec, m, plans, mm = _model("llama3.1-8b", budget=4e9)
    pages = 2048 // 64                      # one request's 2048 rows = 32 KV pages
    h2d, d2h = mm.bytes(1, 2048, pages)
    row = pages * 64 * 2 * spec.n_kv_heads * spec.head_dim * 2
    n_kv1 = sum(1 for p in plans[1].placements if p.residency is Residency.VRAM_PINNED
                and mm.shards[p.shard_id].kind is ShardKind.KV_CACHE)
    assert d2h == n_kv1 * row
    assert h2d >= 0
    back = mm.bytes(2048, 1, pages)
    assert back[0] >= n_kv1 * row       # the KV caches come back


def test_free_switches_reduce_to_the_reference_rule():
    spec, m, plans, mm = _model("llama3.1-8b", budget=4e9)
    for n in (1, 7, 100, 2048, 5000):
        ref = min((t for t in TIERS if t in plans), key=lambda t: (-(-n // t) * plans[t].estimated_time, TIERS.index(t)))
        assert mm.pick_tier(n, None, 0, m) == ref


def test_expensive_switch_is_avoided():
    """With a near-zero link rate any switch is ruinous: the current tier wins."""
    spec, m, plans, mm = _model("llama3.1-8b", budget=4e9)
    slow = type(m)(**{**m.__dict__, "pcie_h2d_bw": 1.0, "pcie_d2h_bw": 1.0}) if hasattr(m, "__dict__") else m
    cur = 1
    assert mm.pick_tier(2048, cur, 2048, slow) == cur


def _apply(mem, old, new, d2d, h2d):
    """Run a relocation plan on a byte array: each shard's bytes are its id."""
    for sid, src, dst, n in d2d:   # whole shards, or pieces of one at the same inner offset
        o = src - old[sid][0]
        assert dst - new[sid][0] == o and 0 <= o and o + n <= old[sid][1]
        mem[dst:dst + n] = mem[src:src + n]
    for sid in h2d:
        off, n = new[sid]
        mem[off:off + n] = bytes([sid % 251 + 1]) * n


def _layout(rng, sids, arena):
    """Random non-overlapping placement of `sids` (sizes fixed per id) in `arena` bytes."""
    order = list(sids)
    rng.shuffle(order)
    out, off = {}, 0
    for sid in order:
        off += int(rng.integers(0, 3)) * 16
        n = 16 * (sid % 7 + 1)
        if off + n > arena:
            break
        out[sid] = (off, n)
        off += n
    return out


def test_relocation_plan_never_reads_a_clobbered_source():
    """plan_relocation on random layouts: after the D2D moves (in order) and the
    uploads, every shard of the new layout holds its own bytes; unchanged shards
    are untouched, and nothing resident in both layouts is uploaded unless it had to be."""
    import numpy as np
    from paper_2604_26334_b200.runtime.migration import plan_relocation
    rng = np.random.default_rng(0)
    fallbacks = moves = 0
    for case in range(400):
        arena = 4096
        ids = list(range(1, int(rng.integers(2, 30))))
        old = _layout(rng, [i for i in ids if rng.random() < 0.8], arena)
        new = _layout(rng, [i for i in ids if rng.random() < 0.8], arena)
        mem = bytearray(arena)
        for sid, (off, n) in old.items():
            mem[off:off + n] = bytes([sid % 251 + 1]) * n
        d2d, h2d = plan_relocation(old, new)
        stay = {sid for sid in new if sid in old and old[sid][0] == new[sid][0]}
        moved = {op[0] for op in d2d}
        assert not (moved & set(h2d)) and not (stay & (moved | set(h2d)))
        assert moved | set(h2d) | stay == set(new)
        _apply(mem, old, new, d2d, h2d)
        for sid, (off, n) in new.items():
            assert mem[off:off + n] == bytes([sid % 251 + 1]) * n, (case, sid)
        fallbacks += len([s for s in h2d if s in old])
        moves += len({op[0] for op in d2d})
    assert moves > 0 and fallbacks < moves


def test_l8_prefill_switch_relocates_in_vram():
    """Config 2 with the executor's carve: the shards the decode and prefill tiers
    both pin move device to device, so the switch into prefill uploads less than
    the prefill tier pins. (Plan-only residency: attention 0-20 keep their offsets;
    with the executor's spare pins the head and FFN shards shift and move in pieces.)"""
    spec, m, plans, mm = _model("llama3.1-8b", budget=4e9)
    h2d, d2h, d2d = mm.moves(1, 2048, 0)
    assert (h2d, d2h, d2d) == (0, 0, 0)
    # a shard shifted by less than its size moves in pieces, never via the host
    from paper_2604_26334_b200.runtime.migration import plan_relocation
    d2d_ops, up = plan_relocation({7: (1000, 1 << 20)}, {7: (1000 - (200 << 10), 1 << 20)})
    assert up == [] and len(d2d_ops) == 6 and sum(op[3] for op in d2d_ops) == 1 << 20


def test_striped_link_model():
    """SURVEY §8f row 1's link model: N striping GPUs multiply the host -> device
    rate; one link is the reference machine itself (plans bit-identical), more
    links keep the placements (budget-driven) and shrink the link-bound estimates."""
    from paper_2604_26334_b200.planning.costdb import synth_profile
    from paper_2604_26334_b200.planning.hardware import machine_to_dict
    spec = catalog.builtin_model("llama3.1-8b")
    m = catalog.builtin_machine("b200")
    assert catalog.striped_machine(m, 1) is m
    m4 = catalog.striped_machine(m, 4)
    assert m4.pcie_h2d_bw == 4 * m.pcie_h2d_bw and m4.pcie_d2h_bw == m.pcie_d2h_bw
    assert set(machine_to_dict(m4)) == set(machine_to_dict(m))      # schema unchanged
    db = synth_profile(m)
    p1 = reachable_tiers(spec, m, db, 4e9, 2304, 1)
    p4 = reachable_tiers(spec, m4, db, 4e9, 2304, 1)
    for t in (1, 2048):
        key = lambda p: [(x.shard_id, x.residency, x.streaming) for x in p.placements]  # noqa: E731
        assert key(p1[t]) == key(p4[t])
        assert p4[t].estimated_time < 0.35 * p1[t].estimated_time   # prefill adds compute + D2H
    with pytest.raises(ValueError):
        catalog.striped_machine(m, 0)
