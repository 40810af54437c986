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
    rows = 2048
    h2d, d2h = mm.bytes(1, 2048, rows)
    row = rows * 1 * 2 * spec.n_kv_heads * spec.head_dim * 2
    n_kv1 = sum(1 for p in plans[1].placements if p.residency is Residency.VRAM_PINNED
                and mm.shards[p.shard_id].kind is ShardKind.KV_CACHE)
    assert d2h == n_kv1 * row
    assert h2d >= 0
    back = mm.bytes(2048, 1, rows)
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
