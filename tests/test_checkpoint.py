"""Checkpoint loading (runtime/checkpoint.py): safetensors parsing, HF-name mapping
onto the shard-contiguous layout (q/k/v concatenation, gate/up interleave, experts,
tied heads), dtype rounding, config.json -> ModelSpec, export round trip. CPU only;
the GPU round trip through Engine is in test_engine_gpu.py."""

import json

import numpy as np
import pytest
import torch

from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.runtime import checkpoint as ck
from paper_2604_26334_b200.runtime.model import WeightLayout, arch_for


def test_bf16_rounding_matches_torch():
    rng = np.random.default_rng(0)
    x = np.concatenate([rng.standard_normal(10000).astype(np.float32) * 10.0 ** rng.integers(-8, 8, 10000),
                        np.array([0.0, -0.0, np.inf, -np.inf, 1e-40, 3.3895314e38], np.float32)])
    want = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ck.bf16_bits(x), want)
    h = rng.standard_normal(1000).astype(np.float16)
    want = torch.from_numpy(h).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ck.bf16_bits(h), want)


def _hf_tensors(spec, arch, rng, tied=False, f32_names=()):
    """Random HF-named tensors for `spec` -> {name: (dtype, shape, array)}."""
    d, hd, h, kv = spec.d_model, spec.head_dim, spec.n_heads, spec.n_kv_heads
    out = {}

    def add(name, shape):
        a = rng.integers(0, 1 << 16, size=shape, dtype=np.uint16)
        a = a & 0x7F7F   # finite bf16 patterns only
        if name in f32_names:
            f = (a.astype(np.uint32) << 16).view(np.float32)
            out[name] = ("F32", shape, f)
        else:
            out[name] = ("BF16", shape, a)

    add("model.embed_tokens.weight", (spec.vocab_size, d))
    for i in range(spec.n_layers):
        p = f"model.layers.{i}."
        add(p + "input_layernorm.weight", (d,))
        add(p + "self_attn.q_proj.weight", (h * hd, d))
        add(p + "self_attn.k_proj.weight", (kv * hd, d))
        add(p + "self_attn.v_proj.weight", (kv * hd, d))
        add(p + "self_attn.o_proj.weight", (d, h * hd))
        if arch.qk_norm:
            add(p + "self_attn.q_norm.weight", (hd,))
            add(p + "self_attn.k_norm.weight", (hd,))
        add(p + "post_attention_layernorm.weight", (d,))
        if spec.moe:
            m = spec.moe
            add(p + "mlp.gate.weight", (m.n_experts, d))
            for e in range(m.n_experts):
                add(p + f"mlp.experts.{e}.gate_proj.weight", (m.expert_ffn_dim, d))
                add(p + f"mlp.experts.{e}.up_proj.weight", (m.expert_ffn_dim, d))
                add(p + f"mlp.experts.{e}.down_proj.weight", (d, m.expert_ffn_dim))
        else:
            add(p + "mlp.gate_proj.weight", (spec.ffn_dim, d))
            add(p + "mlp.up_proj.weight", (spec.ffn_dim, d))
            add(p + "mlp.down_proj.weight", (d, spec.ffn_dim))
    add("model.norm.weight", (d,))
    if not tied:
        add("lm_head.weight", (spec.vocab_size, d))
    return out


def _write(tmp, spec, arch, tensors, shards=2):
    names = list(tensors)
    per = -(-len(names) // shards)
    wm = {}
    for s in range(shards):
        part = {n: tensors[n] for n in names[s * per:(s + 1) * per]}
        fn = f"model-{s + 1:05d}-of-{shards:05d}.safetensors"
        ck.write_safetensors(tmp / fn, part)
        wm.update({n: fn for n in part})
    (tmp / "model.safetensors.index.json").write_text(json.dumps({"weight_map": wm}))
    (tmp / "config.json").write_text(json.dumps(ck.hf_config(spec, arch)))


def _bits(entry):
    dtype, shape, a = entry
    return ck.bf16_bits(a) if dtype == "F32" else a


@pytest.mark.parametrize("model,tied", [("tiny-llama", False), ("tiny-moe", True)])
def test_fill_maps_every_tensor(tmp_path, model, tied):
    spec = catalog.builtin_model(model)
    arch = arch_for(spec)
    rng = np.random.default_rng(1)
    f32 = {"model.layers.0.self_attn.k_proj.weight", "model.norm.weight"}
    tensors = _hf_tensors(spec, arch, rng, tied=tied, f32_names=f32)
    _write(tmp_path, spec, arch, tensors)
    lay = WeightLayout(spec, arch)
    blob = np.zeros(lay.total_bytes, np.uint8)
    emb = np.zeros(lay.embed_bytes, np.uint8)
    c = ck.Checkpoint(tmp_path)
    assert len(c.files) == 2
    ck.fill_from_checkpoint(lay, blob, emb, c)

    def view(sid, name):
        b = lay.blobs[sid]
        t = b.tensors[name]
        o = b.offset + t.offset
        return blob[o:o + t.nbytes].view(np.uint16).reshape(t.rows, t.cols)

    assert np.array_equal(emb.view(np.uint16).reshape(spec.vocab_size, -1),
                          tensors["model.embed_tokens.weight"][2])
    for sid, b in lay.blobs.items():
        i = b.layer
        p = f"model.layers.{i}."
        for name in b.tensors:
            got = view(sid, name)
            leaf = name.split(".", 1)[1] if name.startswith("L") else name
            if leaf == "wqkv":
                want = np.concatenate([_bits(tensors[p + f"self_attn.{x}_proj.weight"]) for x in "qkv"])
            elif leaf == "wgu":
                want = np.empty_like(got)
                want[0::2] = _bits(tensors[p + "mlp.gate_proj.weight"])
                want[1::2] = _bits(tensors[p + "mlp.up_proj.weight"])
            elif leaf.endswith(".wgu"):
                e = int(leaf.split(".")[0][1:])
                want = np.empty_like(got)
                want[0::2] = _bits(tensors[p + f"mlp.experts.{e}.gate_proj.weight"])
                want[1::2] = _bits(tensors[p + f"mlp.experts.{e}.up_proj.weight"])
            elif leaf.endswith(".wdown") and leaf.startswith("e"):
                e = int(leaf.split(".")[0][1:])
                want = _bits(tensors[p + f"mlp.experts.{e}.down_proj.weight"])
            elif name == "lm_head":
                want = _bits(tensors["model.embed_tokens.weight" if tied else "lm_head.weight"])
            else:
                want = _bits(tensors[ck.hf_name(b.tensors[name].init[1])]).reshape(got.shape)
            assert np.array_equal(got, want), name


def test_export_round_trip(tmp_path):
    spec = catalog.builtin_model("tiny-moe")
    arch = arch_for(spec)
    lay = WeightLayout(spec, arch)
    rng = np.random.default_rng(2)
    blob = np.zeros(lay.total_bytes, np.uint8)
    for b in lay.blobs.values():          # random bytes in every tensor, zero padding
        for t in b.tensors.values():
            o = b.offset + t.offset
            blob[o:o + t.nbytes] = rng.integers(0, 256, t.nbytes, dtype=np.uint8)
    emb = rng.integers(0, 256, lay.embed_bytes, dtype=np.uint8)
    files = ck.export_safetensors(lay, blob, emb, tmp_path, max_shard_bytes=1 << 20)
    assert len(files) > 1
    c = ck.Checkpoint(tmp_path)
    spec2, arch2 = ck.spec_from_hf_config(c.config)
    assert (spec2.n_layers, spec2.d_model, spec2.moe, spec2.vocab_size) == \
        (spec.n_layers, spec.d_model, spec.moe, spec.vocab_size)
    assert (arch2.qk_norm, arch2.rms_eps, arch2.rope_theta) == (arch.qk_norm, arch.rms_eps, arch.rope_theta)
    blob2, emb2 = np.zeros_like(blob), np.zeros_like(emb)
    ck.fill_from_checkpoint(WeightLayout(spec2, arch2), blob2, emb2, c)
    assert np.array_equal(blob, blob2) and np.array_equal(emb, emb2)


LLAMA31_8B = {"architectures": ["LlamaForCausalLM"], "hidden_size": 4096, "intermediate_size": 14336,
              "max_position_embeddings": 131072, "model_type": "llama", "num_attention_heads": 32,
              "num_hidden_layers": 32, "num_key_value_heads": 8, "rms_norm_eps": 1e-05,
              "rope_scaling": {"factor": 8.0, "high_freq_factor": 4.0, "low_freq_factor": 1.0,
                               "original_max_position_embeddings": 8192, "rope_type": "llama3"},
              "rope_theta": 500000.0, "tie_word_embeddings": False, "vocab_size": 128256}
QWEN3_30B_A3B = {"architectures": ["Qwen3MoeForCausalLM"], "head_dim": 128, "hidden_size": 2048,
                 "intermediate_size": 6144, "max_position_embeddings": 40960, "model_type": "qwen3_moe",
                 "moe_intermediate_size": 768, "norm_topk_prob": True, "num_attention_heads": 32,
                 "num_experts": 128, "num_experts_per_tok": 8, "num_hidden_layers": 48,
                 "num_key_value_heads": 4, "rms_norm_eps": 1e-06, "rope_theta": 1000000.0,
                 "vocab_size": 151936}


@pytest.mark.parametrize("cfg,preset", [(LLAMA31_8B, "llama3.1-8b"), (QWEN3_30B_A3B, "qwen3-30b-a3b")])
def test_public_configs_match_presets(cfg, preset):
    """The public HF configs of the BASELINE models map to the same ModelSpec /
    Arch the presets hard-code, so a real checkpoint plans exactly like the bench."""
    spec, arch = ck.spec_from_hf_config(cfg, name=preset)
    ref = catalog.builtin_model(preset)
    assert spec == ref
    assert arch == arch_for(ref)


def test_rejects_bad_files(tmp_path):
    (tmp_path / "x.safetensors").write_bytes(b"\x01")
    with pytest.raises(Exception):
        ck.Checkpoint(tmp_path / "x.safetensors")
    with pytest.raises(Exception):
        ck.spec_from_hf_config(dict(LLAMA31_8B, rope_scaling={"rope_type": "yarn", "factor": 4.0}))


@pytest.mark.parametrize("change", [
    {"architectures": ["Qwen2ForCausalLM"], "model_type": "qwen2"},
    {"attention_bias": True}, {"mlp_bias": True}, {"hidden_act": "gelu"},
    {"use_sliding_window": True, "sliding_window": 4096}])
def test_rejects_configs_it_cannot_execute(change):
    """Configs whose numerics this build does not implement are refused instead of
    loading as plain Llama (biases, other activations, sliding windows, other archs)."""
    from paper_2604_26334_b200.planning.faults import SpecError
    with pytest.raises(SpecError):
        ck.spec_from_hf_config(dict(LLAMA31_8B, **change))
    with pytest.raises(SpecError):
        ck.spec_from_hf_config(dict(QWEN3_30B_A3B, mlp_only_layers=[0]))


def test_rejects_checkpoint_with_unconsumed_tensors(tmp_path):
    """A q_proj.bias (a Qwen2-style checkpoint) is a tensor the layout does not consume:
    loading fails loudly instead of dropping it."""
    from paper_2604_26334_b200.planning.faults import FormatError
    spec = catalog.builtin_model("tiny-llama")
    arch = arch_for(spec)
    tensors = _hf_tensors(spec, arch, np.random.default_rng(2), tied=False, f32_names=set())
    tensors["model.layers.0.self_attn.q_proj.bias"] = ("BF16", (spec.n_heads * spec.head_dim,),
                                                       np.zeros(spec.n_heads * spec.head_dim, np.uint16))
    _write(tmp_path, spec, arch, tensors, shards=1)
    lay = WeightLayout(spec, arch)
    with pytest.raises(FormatError, match="q_proj.bias"):
        ck.fill_from_checkpoint(lay, np.zeros(lay.total_bytes, np.uint8), np.zeros(lay.embed_bytes, np.uint8),
                                ck.Checkpoint(tmp_path))


# -- GGUF (runtime/gguf.py) ---------------------------------------------------------

def test_gguf_rope_permutation_is_llama_cpp_order():
    """llama.cpp stores each llama q/k head with rotary pairs adjacent: HF rows
    (0, 1, 2, 3) of a 4-dim head are stored as (0, 2, 1, 3); unpermute inverts it."""
    from paper_2604_26334_b200.runtime import gguf
    w = np.arange(8, dtype=np.uint16).reshape(8, 1)          # 2 heads x hd 4
    p = gguf.permute_rope_rows(w, 2)
    assert p[:, 0].tolist() == [0, 2, 1, 3, 4, 6, 5, 7]
    assert np.array_equal(gguf.unpermute_rope_rows(p, 2), w)


@pytest.mark.parametrize("model", ["tiny-llama", "tiny-moe", "llama3.1-8b"])
def test_gguf_round_trip_fills_identical_blob(tmp_path, model):
    """safetensors -> blob -> write_gguf -> GgufCheckpoint -> blob is byte-identical;
    the GGUF config yields the same ModelSpec and Arch (incl. llama3 rope scaling as
    rope_freqs, stacked experts, permuted llama q/k, F32 norms)."""
    from paper_2604_26334_b200.runtime import gguf
    from paper_2604_26334_b200.runtime.model import Arch
    spec = catalog.builtin_model(model)
    if model == "llama3.1-8b":   # the real shapes, 2 layers
        import dataclasses
        spec = dataclasses.replace(spec, n_layers=2, vocab_size=4096)
    arch = arch_for(catalog.builtin_model(model))
    rng = np.random.default_rng(3)
    tensors = _hf_tensors(spec, arch, rng)
    _write(tmp_path, spec, arch, tensors)
    lay = WeightLayout(spec, arch)
    blob = np.zeros(lay.total_bytes, np.uint8)
    emb = np.zeros(lay.embed_bytes, np.uint8)
    ck.fill_from_checkpoint(lay, blob, emb, ck.Checkpoint(tmp_path))
    path = tmp_path / "m.gguf"
    gguf.write_gguf(path, lay, blob, emb, arch)
    g = ck.open_checkpoint(path)
    assert isinstance(g, gguf.GgufCheckpoint)
    spec2, arch2 = ck.spec_from_hf_config(g.config)
    for f in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim", "vocab_size", "moe"):
        assert getattr(spec2, f) == getattr(spec, f), f
    assert (spec2.ffn_dim == spec.ffn_dim) or spec.moe
    assert isinstance(arch2, Arch) and arch2.qk_norm == arch.qk_norm
    assert arch2.rope_theta == pytest.approx(arch.rope_theta) and arch2.rope_scaling == arch.rope_scaling
    blob2 = np.zeros_like(blob)
    emb2 = np.zeros_like(emb)
    ck.fill_from_checkpoint(lay, blob2, emb2, g)
    assert np.array_equal(blob2, blob) and np.array_equal(emb2, emb)
    if arch.qk_norm is False:   # llama: q rows really are stored permuted in the file
        hd, h = spec.head_dim, spec.n_heads
        raw = np.asarray(g.file.array("blk.0.attn_q.weight"))
        hf = tensors["model.layers.0.self_attn.q_proj.weight"][2]
        assert not np.array_equal(raw, hf)
        assert np.array_equal(raw, gguf.permute_rope_rows(hf, h))


def test_gguf_rejects_bad_files(tmp_path):
    from paper_2604_26334_b200.planning.faults import FormatError, SpecError
    from paper_2604_26334_b200.runtime import gguf
    p = tmp_path / "x.gguf"
    p.write_bytes(b"NOPE" + b"\0" * 64)
    with pytest.raises(FormatError):
        gguf.GgufFile(p)
    import struct
    # a valid header whose architecture is not supported
    k, v = b"general.architecture", b"gpt2"
    p.write_bytes(b"GGUF" + struct.pack("<IQQ", 3, 0, 1) + struct.pack("<Q", len(k)) + k +
                  struct.pack("<IQ", 8, len(v)) + v + b"\0" * 32)
    with pytest.raises(SpecError):
        gguf.GgufCheckpoint(p)


def test_exponent_coding_round_trip():
    """runtime/wcomp.py: 12-bit exponent-coded rows decode to the exact bf16 bits,
    escapes (zeros, denormals, inf/nan, far exponents) included, each row with its own
    base exponent (a heavy-tailed head row needs no escapes); a matrix with a row of
    more than MAX_ESCAPES escapes is refused (streams as bf16)."""
    from oracle import model_ref as M
    from paper_2604_26334_b200.runtime import wcomp
    bits = M.bf16_bits(0, "L0.w_gate", 256, 512).copy()
    bits[0, :4] = [0x0000, 0x8000, 0x0001, 0x7F80]       # +0, -0, denormal, inf
    bits[1, 7] = 0x7FC1                                  # nan
    bits[2, 9] = 0x4700                                  # 32768, far above the window
    res = wcomp.encode(bits)
    assert res is not None
    coded, tb = res
    assert coded.shape == (256, 768 + tb) and coded.dtype == np.uint8 and tb % 16 == 0
    assert np.array_equal(wcomp.decode(coded, 512), bits)
    n_esc = (coded[:, 768:].copy().view(np.uint32)[:, 0] >> 8).sum()
    assert n_esc < 1e-3 * bits.size + 1100               # row 2: everything below 2^15 / 2^14
    assert wcomp._trailer_or_none(bits) == tb
    head = M.bf16_bits(0, "lm_head", 512, 512)           # heavy-tailed rows: own windows
    c2, tb2 = wcomp.encode(head)
    assert np.array_equal(wcomp.decode(c2, 512), head) and tb2 <= 32
    many = bits.copy()
    many[5, :100] = 0x0001                               # 100 denormals in one row
    assert wcomp.encode(many) is None and wcomp._trailer_or_none(many) is None
    with pytest.raises(ValueError):
        wcomp.encode(bits[:, :511])
