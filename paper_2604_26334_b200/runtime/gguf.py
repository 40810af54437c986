"""GGUF checkpoints -> the shard-contiguous pinned blob.

The paper runs its models from GGUF files (`PAPER.md:789`); this module reads
the unquantised subset of that format (F32 / F16 / BF16 tensors) and presents it
through the same interface as `checkpoint.Checkpoint` — an HF-style `config`
dict, `has(hf_name)` and `bf16(hf_name, shape)` — so `fill_from_checkpoint`,
`Engine(None, checkpoint="model.gguf")` and the planner see no difference.

Format (GGUF v3, little endian): magic "GGUF", version u32, tensor count u64,
metadata count u64; metadata as (string key, u32 type, value); tensor infos as
(string name, u32 n_dims, u64 ne[n_dims] innermost first, u32 ggml type, u64
offset); then the data section at the next multiple of `general.alignment`
(default 32). A PyTorch weight [out, in] is stored with ne = [in, out].

Conventions of llama.cpp-produced files that this loader undoes:
* tensor names `token_embd`, `blk.N.attn_q`, `ffn_gate_exps`, … (`GGUF_NAMES`);
* MoE experts stacked per layer in one 3-D tensor per projection;
* for the `llama` architecture the q/k projection rows of every head are
  permuted so that rotary pairs are adjacent (llama.cpp's rope pairs dims
  2i, 2i+1; the HF layout and this build's kernels pair i, i + hd/2) —
  `unpermute_rope_rows` restores the HF order; `qwen3*` files are unpermuted;
* Llama-3 rope scaling travels as a `rope_freqs.weight` tensor of per-pair
  factors; it is accepted when it equals the factors of the standard llama3
  parameters (`model.LLAMA3_SCALING`) and rejected otherwise.

`write_gguf` produces such a file from a filled host blob (round-trip tests and
a way to hand this build's random-init models to GGUF tooling).
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from ..planning.faults import FormatError, SpecError
from .checkpoint import _copy_jobs, bf16_bits, hf_name
from .model import LLAMA3_SCALING, Arch, WeightLayout, rope_inv_freq

GGUF_MAGIC = b"GGUF"
T_F32, T_F16, T_BF16 = 0, 1, 30
_NP = {T_F32: np.float32, T_F16: np.float16, T_BF16: np.uint16}
_ITEM = {T_F32: 4, T_F16: 2, T_BF16: 2}
# metadata value types
V_U8, V_I8, V_U16, V_I16, V_U32, V_I32, V_F32, V_BOOL, V_STR, V_ARR, V_U64, V_I64, V_F64 = range(13)
_SCALAR = {V_U8: "<B", V_I8: "<b", V_U16: "<H", V_I16: "<h", V_U32: "<I", V_I32: "<i", V_F32: "<f",
           V_BOOL: "<?", V_U64: "<Q", V_I64: "<q", V_F64: "<d"}

# HF leaf name -> GGUF leaf name, per layer
GGUF_NAMES = {
    "input_layernorm.weight": "attn_norm.weight",
    "post_attention_layernorm.weight": "ffn_norm.weight",
    "self_attn.q_proj.weight": "attn_q.weight",
    "self_attn.k_proj.weight": "attn_k.weight",
    "self_attn.v_proj.weight": "attn_v.weight",
    "self_attn.o_proj.weight": "attn_output.weight",
    "self_attn.q_norm.weight": "attn_q_norm.weight",
    "self_attn.k_norm.weight": "attn_k_norm.weight",
    "mlp.gate_proj.weight": "ffn_gate.weight",
    "mlp.up_proj.weight": "ffn_up.weight",
    "mlp.down_proj.weight": "ffn_down.weight",
    "mlp.gate.weight": "ffn_gate_inp.weight",
}
_EXPERT_NAMES = {"gate_proj": "ffn_gate_exps.weight", "up_proj": "ffn_up_exps.weight",
                 "down_proj": "ffn_down_exps.weight"}


def unpermute_rope_rows(w: np.ndarray, n_heads: int) -> np.ndarray:
    """llama.cpp row order (per head: pairs (2i, 2i+1) adjacent) -> HF order
    (pairs (i, i + hd/2)). w: [n_heads * hd, cols]."""
    rows, cols = w.shape
    hd = rows // n_heads
    return w.reshape(n_heads, hd // 2, 2, cols).swapaxes(1, 2).reshape(rows, cols)


def permute_rope_rows(w: np.ndarray, n_heads: int) -> np.ndarray:
    """Inverse of `unpermute_rope_rows` (HF -> llama.cpp order)."""
    rows, cols = w.shape
    hd = rows // n_heads
    return w.reshape(n_heads, 2, hd // 2, cols).swapaxes(1, 2).reshape(rows, cols)


def llama3_rope_factors(theta: float, head_dim: int, scaling: dict) -> np.ndarray:
    """Per-pair divisors of the base inverse frequencies (llama.cpp's rope_freqs)."""
    base = rope_inv_freq(Arch(rope_theta=theta), head_dim)
    scaled = rope_inv_freq(Arch(rope_theta=theta, rope_scaling=scaling), head_dim)
    return (base / scaled).astype(np.float32)


class GgufFile:
    """Metadata, tensor directory and a memory map of one .gguf file."""

    def __init__(self, path):
        self.path = str(path)
        self._mm = np.memmap(self.path, dtype=np.uint8, mode="r")
        self._pos = 0
        if bytes(self._mm[:4]) != GGUF_MAGIC:
            raise FormatError(f"{self.path}: not a GGUF file")
        self._pos = 4
        self.version = self._u("<I")
        if self.version not in (2, 3):
            raise FormatError(f"{self.path}: GGUF version {self.version} unsupported")
        n_tensors, n_kv = self._u("<Q"), self._u("<Q")
        self.meta = {}
        for _ in range(n_kv):
            key = self._str()
            self.meta[key] = self._value(self._u("<I"))
        self.tensors = {}
        for _ in range(n_tensors):
            name = self._str()
            nd = self._u("<I")
            ne = [self._u("<Q") for _ in range(nd)]
            ttype = self._u("<I")
            off = self._u("<Q")
            if ttype not in _NP:
                raise FormatError(f"{self.path}: tensor {name} has quantised/unsupported type {ttype}")
            self.tensors[name] = (tuple(reversed(ne)), ttype, off)   # numpy (row-major) shape
        align = int(self.meta.get("general.alignment", 32))
        self.data_start = -(-self._pos // align) * align
        size = len(self._mm)
        for name, (shape, ttype, off) in self.tensors.items():
            end = self.data_start + off + int(np.prod(shape, dtype=np.int64)) * _ITEM[ttype]
            if off % align or end > size:
                raise FormatError(f"{self.path}: tensor {name} lies outside the data section")

    def _u(self, fmt):
        n = struct.calcsize(fmt)
        (v,) = struct.unpack(fmt, bytes(self._mm[self._pos:self._pos + n]))
        self._pos += n
        return v

    def _str(self):
        n = self._u("<Q")
        s = bytes(self._mm[self._pos:self._pos + n]).decode("utf-8")
        self._pos += n
        return s

    def _value(self, vtype):
        if vtype in _SCALAR:
            return self._u(_SCALAR[vtype])
        if vtype == V_STR:
            return self._str()
        if vtype == V_ARR:
            etype, n = self._u("<I"), self._u("<Q")
            return [self._value(etype) for _ in range(n)]
        raise FormatError(f"{self.path}: metadata value type {vtype}")

    def array(self, name: str) -> np.ndarray:
        shape, ttype, off = self.tensors[name]
        n = int(np.prod(shape, dtype=np.int64)) * _ITEM[ttype]
        raw = self._mm[self.data_start + off:self.data_start + off + n]
        return raw.view(_NP[ttype]).reshape(shape)


class GgufCheckpoint:
    """A .gguf file behind `checkpoint.Checkpoint`'s interface (HF names)."""

    def __init__(self, path):
        self.file = GgufFile(path)
        self.files = [self.file]
        m = self.file.meta
        arch = m.get("general.architecture")
        if arch not in ("llama", "qwen3", "qwen3moe"):
            raise SpecError(f"{path}: GGUF architecture {arch!r} is not supported")
        self.arch_name = arch
        g = lambda key, default=None: m.get(f"{arch}.{key}", default)  # noqa: E731
        d, heads = g("embedding_length"), g("attention.head_count")
        vocab = self.file.tensors["token_embd.weight"][0][0]
        cfg = {"architectures": [{"llama": "LlamaForCausalLM", "qwen3": "Qwen3ForCausalLM",
                                  "qwen3moe": "Qwen3MoeForCausalLM"}[arch]],
               "model_type": {"llama": "llama", "qwen3": "qwen3", "qwen3moe": "qwen3_moe"}[arch],
               "_name_or_path": m.get("general.name", Path(path).stem),
               "hidden_size": d, "num_hidden_layers": g("block_count"), "num_attention_heads": heads,
               "num_key_value_heads": g("attention.head_count_kv", heads),
               "head_dim": g("attention.key_length", d // heads),
               "intermediate_size": g("feed_forward_length", 0) or g("expert_feed_forward_length"),
               "vocab_size": vocab, "max_position_embeddings": g("context_length", 4096),
               "rms_norm_eps": g("attention.layer_norm_rms_epsilon", 1e-5),
               "rope_theta": g("rope.freq_base", 10000.0)}
        if g("expert_count"):
            cfg.update(num_experts=g("expert_count"), num_experts_per_tok=g("expert_used_count"),
                       moe_intermediate_size=g("expert_feed_forward_length"), norm_topk_prob=True)
        if "rope_freqs.weight" in self.file.tensors:
            got = np.asarray(self.file.array("rope_freqs.weight"), np.float32).reshape(-1)
            want = llama3_rope_factors(cfg["rope_theta"], cfg["head_dim"], LLAMA3_SCALING)
            if got.shape != want.shape or not np.allclose(got, want, rtol=1e-6, atol=0):
                raise SpecError(f"{path}: rope_freqs are not the standard llama3 scaling")
            cfg["rope_scaling"] = dict(LLAMA3_SCALING, rope_type="llama3")
        self.config = cfg

    def _locate(self, name: str):
        """HF name -> (gguf tensor, expert index or None, rope heads to unpermute or 0)."""
        if name == "model.embed_tokens.weight":
            return "token_embd.weight", None, 0
        if name == "model.norm.weight":
            return "output_norm.weight", None, 0
        if name == "lm_head.weight":
            return "output.weight", None, 0
        if not name.startswith("model.layers."):
            return None, None, 0
        i, leaf = name[len("model.layers."):].split(".", 1)
        if leaf.startswith("mlp.experts."):
            e, proj, _ = leaf[len("mlp.experts."):].split(".")
            return f"blk.{i}.{_EXPERT_NAMES[proj]}", int(e), 0
        g = GGUF_NAMES.get(leaf)
        if g is None:
            return None, None, 0
        heads = 0
        if self.arch_name == "llama" and leaf in ("self_attn.q_proj.weight", "self_attn.k_proj.weight"):
            heads = self.config["num_attention_heads"] if "q_proj" in leaf else self.config["num_key_value_heads"]
        return f"blk.{i}.{g}", None, heads

    def has(self, name: str) -> bool:
        t, _, _ = self._locate(name)
        return t is not None and t in self.file.tensors

    def bf16(self, name: str, shape: tuple) -> np.ndarray:
        t, expert, heads = self._locate(name)
        if t is None or t not in self.file.tensors:
            raise FormatError(f"checkpoint has no tensor {name}")
        a = self.file.array(t)
        if expert is not None:
            a = a[expert]
        n = int(np.prod(shape, dtype=np.int64))
        if a.size != n:
            raise FormatError(f"{name}: GGUF shape {a.shape} does not fit {shape}")
        ttype = self.file.tensors[t][1]
        bits = a.reshape(shape) if ttype == T_BF16 else bf16_bits(a).reshape(shape)
        if heads:
            bits = unpermute_rope_rows(np.asarray(bits), heads)
        return bits


def _gguf_name(hf: str, arch: str, n_heads: int, n_kv: int):
    """HF name -> (GGUF name, expert index or None, heads to permute or 0)."""
    if hf == "model.embed_tokens.weight":
        return "token_embd.weight", None, 0
    if hf == "model.norm.weight":
        return "output_norm.weight", None, 0
    if hf == "lm_head.weight":
        return "output.weight", None, 0
    i, leaf = hf[len("model.layers."):].split(".", 1)
    if leaf.startswith("mlp.experts."):
        e, proj, _ = leaf[len("mlp.experts."):].split(".")
        return f"blk.{i}.{_EXPERT_NAMES[proj]}", int(e), 0
    heads = 0
    if arch == "llama" and leaf == "self_attn.q_proj.weight":
        heads = n_heads
    elif arch == "llama" and leaf == "self_attn.k_proj.weight":
        heads = n_kv
    return f"blk.{i}.{GGUF_NAMES[leaf]}", None, heads


def write_gguf(path, layout: WeightLayout, blob: np.ndarray, embed: np.ndarray, arch: Arch,
               name: str | None = None, alignment: int = 32) -> int:
    """Write a filled host blob (uint8) + embedding table as a GGUF v3 file with
    llama.cpp conventions: matrices BF16, norms F32, experts stacked, llama q/k
    rows rope-permuted, llama3 scaling as rope_freqs. Returns the file size."""
    spec = layout.spec
    g_arch = "qwen3moe" if spec.moe else ("qwen3" if arch.qk_norm else "llama")
    tensors: dict = {}
    experts: dict = {}
    tensors["token_embd.weight"] = (T_BF16, embed.view(np.uint16).reshape(spec.vocab_size, spec.d_model))
    for logical, dst, rows, cols, mode in _copy_jobs(layout, False):
        if mode == "plain":
            a = blob[dst:dst + rows * cols * 2].view(np.uint16).reshape(rows, cols)
        else:
            full = blob[dst:dst + 2 * rows * cols * 2].view(np.uint16).reshape(2 * rows, cols)
            a = full[mode[1]::2]
        gname, expert, heads = _gguf_name(hf_name(logical), g_arch, spec.n_heads, spec.n_kv_heads)
        if heads:
            a = permute_rope_rows(np.asarray(a), heads)
        if expert is not None:
            experts.setdefault(gname, {})[expert] = np.asarray(a)
        elif rows == 1:   # norms as F32 (exact: bf16 -> f32)
            tensors[gname] = (T_F32, (np.asarray(a).astype(np.uint32) << 16).view(np.float32).reshape(-1))
        else:
            tensors[gname] = (T_BF16, np.asarray(a))
    for gname, per in experts.items():
        tensors[gname] = (T_BF16, np.stack([per[e] for e in range(len(per))]))
    if arch.rope_scaling:
        tensors["rope_freqs.weight"] = (T_F32, llama3_rope_factors(arch.rope_theta, spec.head_dim,
                                                                   arch.rope_scaling))
    meta = [("general.architecture", V_STR, g_arch), ("general.name", V_STR, name or spec.name),
            ("general.alignment", V_U32, alignment),
            (f"{g_arch}.block_count", V_U32, spec.n_layers),
            (f"{g_arch}.context_length", V_U32, spec.max_context),
            (f"{g_arch}.embedding_length", V_U32, spec.d_model),
            (f"{g_arch}.feed_forward_length", V_U32, spec.ffn_dim),
            (f"{g_arch}.attention.head_count", V_U32, spec.n_heads),
            (f"{g_arch}.attention.head_count_kv", V_U32, spec.n_kv_heads),
            (f"{g_arch}.attention.key_length", V_U32, spec.head_dim),
            (f"{g_arch}.attention.value_length", V_U32, spec.head_dim),
            (f"{g_arch}.attention.layer_norm_rms_epsilon", V_F32, arch.rms_eps),
            (f"{g_arch}.rope.freq_base", V_F32, arch.rope_theta)]
    if spec.moe:
        meta += [(f"{g_arch}.expert_count", V_U32, spec.moe.n_experts),
                 (f"{g_arch}.expert_used_count", V_U32, spec.moe.top_k),
                 (f"{g_arch}.expert_feed_forward_length", V_U32, spec.moe.expert_ffn_dim)]

    def s(x: str) -> bytes:
        b = x.encode()
        return struct.pack("<Q", len(b)) + b

    head = bytearray(GGUF_MAGIC + struct.pack("<IQQ", 3, len(tensors), len(meta)))
    for key, vt, v in meta:
        head += s(key) + struct.pack("<I", vt) + (s(v) if vt == V_STR else struct.pack(_SCALAR[vt], v))
    offsets, off = {}, 0
    for gname, (tt, a) in tensors.items():
        offsets[gname] = off
        off += -(-a.size * _ITEM[tt] // alignment) * alignment
    for gname, (tt, a) in tensors.items():
        head += s(gname) + struct.pack("<I", a.ndim) + b"".join(struct.pack("<Q", n) for n in reversed(a.shape))
        head += struct.pack("<IQ", tt, offsets[gname])
    head += b"\0" * (-len(head) % alignment)
    with open(path, "wb") as fh:
        fh.write(head)
        for gname, (tt, a) in tensors.items():
            data = np.ascontiguousarray(a).tobytes()
            fh.write(data)
            fh.write(b"\0" * (-len(data) % alignment))
    return Path(path).stat().st_size
