"""End-to-end parity of the streaming executor against the fp32 oracle.

Tiny config (BASELINE.json configs[0]): 4 layers, d=512, 8 heads, prompt
128 + 32 decode, VRAM budget = 50 % of plan weights — the plan mixes
pinned, scratch-packed, streamed and CPU-placed (zero-copy) shards. Greedy
tokens must be identical; logits within max|d| / max|ref| <= 2e-2
(north_star tolerance).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from paper_2604_26334_b200.planning import catalog  # noqa: E402
from paper_2604_26334_b200.planning.graph import total_model_bytes  # noqa: E402


@pytest.fixture(scope="module")
def tiny():
    return catalog.builtin_model("tiny-llama")


@pytest.fixture(scope="module")
def oracle(tiny):
    from oracle.model_ref import RefModel, hp_from_spec
    from paper_2604_26334_b200.runtime.model import arch_for
    return RefModel(hp_from_spec(tiny, arch_for(tiny)), seed=0)


def _prompt(n, V, seed=0):
    return np.random.default_rng(seed).integers(0, V, n).astype(np.int32)


@pytest.mark.parametrize("frac", [0.5, 0.25, 1.5])
def test_tiny_generate_matches_oracle(tiny, oracle, frac):
    from paper_2604_26334_b200.runtime.engine import Engine
    budget = frac * total_model_bytes(tiny)
    eng = Engine(tiny, budget_bytes=budget, context_len=160)
    prompt = _prompt(128, tiny.vocab_size)
    res = eng.generate([prompt], gen_len=32)
    got = res.tokens[0]
    want, ref_logits = oracle.greedy(prompt, 32)
    kinds = {t: p.kind.value for t, p in eng.plans.items()}
    eng.close()
    assert len(got) == 32
    assert np.array_equal(got, want), (frac, kinds, got, want)


def test_host_weights_bit_exact_vs_oracle(tiny):
    from oracle import model_ref
    from paper_2604_26334_b200.runtime.model import HostWeights, arch_for
    hw = HostWeights(tiny, arch_for(tiny))
    hw.generate()
    lay = hw.layout
    attn0 = [sid for sid, b in lay.blobs.items() if b.layer == 0 and b.kind.value == "attention"][0]
    wqkv = hw.host_view(attn0, "L0.wqkv")
    h, kv, hd, d = tiny.n_heads, tiny.n_kv_heads, tiny.head_dim, tiny.d_model
    np.testing.assert_array_equal(wqkv[: h * hd], model_ref.bf16_bits(0, "L0.wq", h * hd, d))
    np.testing.assert_array_equal(wqkv[h * hd:(h + kv) * hd], model_ref.bf16_bits(0, "L0.wk", kv * hd, d))
    ffn0 = [sid for sid, b in lay.blobs.items() if b.layer == 0 and b.kind.value == "ffn"][0]
    np.testing.assert_array_equal(hw.host_view(ffn0, "L0.wgu"),
                                  model_ref.interleaved_bits(0, "L0.w_gate", "L0.w_up", tiny.ffn_dim, d))
    np.testing.assert_array_equal(hw.embed_view(), model_ref.bf16_bits(0, "embed", tiny.vocab_size, d))
    hw.close()


def test_decode_logits_within_tolerance(tiny, oracle):
    from paper_2604_26334_b200.runtime.engine import Engine
    eng = Engine(tiny, budget_bytes=0.5 * total_model_bytes(tiny), context_len=160)
    prompt = _prompt(40, tiny.vocab_size, seed=3)
    res = eng.generate([prompt], gen_len=4)
    gpu_last = eng.executor.logits_host(1)[0]
    tf = oracle.teacher_forced(prompt, res.tokens[0]).numpy()
    eng.close()
    ref_last = tf[-1]
    err = np.abs(gpu_last - ref_last).max() / np.abs(ref_last).max()
    assert err <= 2e-2, err


def test_arena_refuses_over_budget(tiny):
    from paper_2604_26334_b200.runtime.arena import ArenaExhausted, VramArena
    a = VramArena(1 << 20)
    a.alloc_low("x", 700 << 10)
    with pytest.raises(ArenaExhausted):
        a.alloc_high("y", 400 << 10)
