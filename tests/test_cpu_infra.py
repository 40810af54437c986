"""CPU-side checks: oracle known answers, host layout, C-ABI exports, tier reachability."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.planning.graph import build_shards, total_model_bytes
from paper_2604_26334_b200.planning.placement import reachable_tiers
from paper_2604_26334_b200.planning.costdb import synth_profile

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _py_value(seed, idx, scale, bias):
    """Pure-Python restatement of one element of the initialiser (small cases)."""
    m = (1 << 64) - 1
    z = seed ^ ((idx * 0x9E3779B97F4A7C15) & m)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    z ^= z >> 31
    u = np.float32((z >> 40) * (1.0 / 16777216.0))
    w = np.float32(np.float32(2.0) * u - np.float32(1.0))
    v = np.float64(w) * np.float64(np.float32(scale)) + np.float64(np.float32(bias))
    f = np.float32(v)   # fmaf: single rounding of the exact product-sum
    b = int(f.view(np.uint32))
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFFFFFF
    return b >> 16


def test_oracle_initialiser_matches_python_restatement():
    from oracle import model_ref
    bits = model_ref.bf16_bits(7, "L0.wq", 4, 64)
    sc, bi = model_ref.scale_bias("L0.wq", 64)
    sd = model_ref.seed_of(7, "L0.wq")
    want = np.array([_py_value(sd, i, sc, bi) for i in range(4 * 64)], np.uint16).reshape(4, 64)
    np.testing.assert_array_equal(bits, want)
    gu = model_ref.interleaved_bits(7, "L0.w_gate", "L0.w_up", 3, 64)
    np.testing.assert_array_equal(gu[0::2], model_ref.bf16_bits(7, "L0.w_gate", 3, 64))
    np.testing.assert_array_equal(gu[1::2], model_ref.bf16_bits(7, "L0.w_up", 3, 64))


def _py_head_row_scale(seed, row):
    m = (1 << 64) - 1
    z = (seed ^ 0xD1B54A32D192ED03) ^ ((row * 0x9E3779B97F4A7C15) & m)
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & m
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & m
    z ^= z >> 31
    u = np.float32((np.float32(z >> 40) + np.float32(0.5)) * np.float32(1.0 / 16777216.0))
    s = np.float32(np.float32(1.0) / np.sqrt(u, dtype=np.float32))   # IEEE sqrt and div
    return min(s, np.float32(64.0))


def test_oracle_head_init_matches_python_restatement():
    """The output head's heavy-tailed rows (margin-robust init): every element is the
    uniform value with scale * s_row, s_row = min(u^-1/2, 64), all IEEE-rounded ops."""
    from oracle import model_ref
    rows, cols = 6, 64
    bits = model_ref.bf16_bits(3, "lm_head", rows, cols)
    sc, _ = model_ref.scale_bias("lm_head", cols)
    sd = model_ref.seed_of(3, "lm_head")
    want = np.array([_py_value(sd, i, np.float32(np.float32(sc) * _py_head_row_scale(sd, i // cols)), 0.0)
                     for i in range(rows * cols)], np.uint16).reshape(rows, cols)
    np.testing.assert_array_equal(bits, want)
    # heavy tail: over many rows a few are scaled far above the median
    big = model_ref.weight(0, "lm_head", 4096, 64).abs().amax(1).numpy()
    assert big.max() > 20 * np.median(big)


def test_oracle_norm_init_range():
    from oracle import model_ref
    w = model_ref.weight(0, "L3.attn_norm", 1, 4096).numpy()
    assert 0.89 <= w.min() and w.max() <= 1.11


def test_rope_table_matches_oracle():
    from oracle import model_ref
    from paper_2604_26334_b200.runtime.model import arch_for, rope_table, rope_inv_freq
    spec = catalog.builtin_model("llama3.1-8b")
    arch = arch_for(spec)
    a = rope_inv_freq(arch, 128)
    b = model_ref.inv_freq(arch.rope_theta, 128, arch.rope_scaling)
    np.testing.assert_allclose(a, b, rtol=1e-15)
    tab = rope_table(arch, 128, 64)
    ang = np.arange(64)[:, None] * b[None, :]
    np.testing.assert_array_equal(tab[..., 0], np.cos(ang).astype(np.float32))


def test_weight_layout_covers_plan_bytes():
    from paper_2604_26334_b200.runtime.model import WeightLayout, arch_for
    for name in ("tiny-llama", "llama3.1-8b", "llama3.3-70b"):
        spec = catalog.builtin_model(name)
        lay = WeightLayout(spec, arch_for(spec))
        shards = {s.id: s for s in build_shards(spec, 0)}
        for sid, blob in lay.blobs.items():
            # physical = plan weight bytes + norm vectors + 256-B alignment padding
            extra = blob.nbytes - shards[sid].weight_bytes
            assert 0 <= extra <= 4 * 256 + 4 * spec.d_model, (name, sid, extra)
        assert lay.total_bytes >= total_model_bytes(spec)


def test_tiny_config_reachable_tiers():
    spec = catalog.builtin_model("tiny-llama")
    machine = catalog.builtin_machine("b200")
    budget = 0.5 * total_model_bytes(spec)
    plans = reachable_tiers(spec, machine, synth_profile(machine), budget, 160)
    assert set(plans) == {1, 4, 16, 32, 64, 512, 1024, 2048, 4096}


def test_header_exports_match_binding():
    from paper_2604_26334_b200.runtime import lib as L
    header = open(os.path.join(REPO, "include", "pshard.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char\*)\s+(ps_\w+)\(", header, re.M))
    assert declared == set(L.EXPORTED), declared ^ set(L.EXPORTED)


def test_library_loads_and_exports_every_symbol():
    from paper_2604_26334_b200.runtime import lib as L
    if not os.path.exists(L.LIB_PATH):
        pytest.skip("libpshard.so not built (run __graft_entry__.build())")
    lib = ctypes.CDLL(L.LIB_PATH)
    for name in L.EXPORTED:
        assert hasattr(lib, name), name
    assert lib.ps_abi_version() == 1


def test_speculative_fetch_settlement(monkeypatch):
    """Executor.settle (host bookkeeping of speculative expert prefetch, no GPU): a pass's
    link bytes become what the fetcher copied (misses + predictions) once its job is
    processed; routed experts that were not copied count as prefetch hits; jobs the
    fetcher has not processed yet (-1) stay pending."""
    from paper_2604_26334_b200.runtime import executor as X
    copied = {10: 8 * 100, 11: 6 * 100 + 2 * 90, 12: -1}   # seq -> bytes (-1: not processed)

    def fake_call(name, *args):
        assert name == "ps_fetcher_seq_bytes"
        args[2]._obj.value = copied[args[1]]
        return 0
    monkeypatch.setattr(X.L, "call", fake_call)
    ex = X.Executor.__new__(X.Executor)
    ex.fetcher = 1
    st = X.PassStats(tier=1, T=1, bytes_streamed=3 * 800)
    # (seq, bytes counted at enqueue, expert bytes, prediction bytes, routed experts with a
    # prediction set, predictions made)
    st.fetch_seqs = [(10, 800, 100, 0, 0, 0), (11, 800, 100, 2 * 90, 8, 2), (12, 800, 100, 2 * 90, 8, 2)]
    ex._unsettled = [st]
    ex.settle()
    assert st.bytes_streamed == 3 * 800 + (800 - 800) + (780 - 800)
    assert (st.spec_routed, st.spec_hits) == (8, 2)
    assert st.fetch_seqs == [(12, 800, 100, 180, 8, 2)] and ex._unsettled == [st]
    assert (st.spec_predicted, st.spec_pred_bytes) == (2, 180)
    copied[12] = 5 * 100 + 2 * 90
    ex.settle()
    assert st.bytes_streamed == 3 * 800 - 20 - 120
    assert (st.spec_routed, st.spec_hits) == (16, 5)
    assert (st.spec_predicted, st.spec_pred_bytes) == (4, 360)
    assert not st.fetch_seqs and ex._unsettled == []
