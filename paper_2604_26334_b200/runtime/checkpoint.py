"""Real checkpoints: Hugging Face safetensors -> the shard-contiguous pinned blob.

SURVEY.md §8f row 4. The reference has no weights at all (`pkg/README.md:20-22`);
the paper loads GGUF files into llama.cpp (`PAPER.md:789`). This build's
on-disk format is the one public Llama / Qwen3 checkpoints ship in:
`config.json` + `*.safetensors` (optionally sharded with
`model.safetensors.index.json`). Loading maps each HF tensor onto the
executor's layout (`runtime/model.py`): q/k/v rows concatenated into `wqkv`,
gate/up rows interleaved into `wgu` (so SwiGLU runs in the producing
kernel's epilogue), experts laid out expert-contiguous inside their MoE
group, norms inside their shard. BF16 tensors are copied byte for byte;
F16 / F32 tensors are rounded to bf16 (round-to-nearest-even). Nothing
touches the GPU: the blob is filled through numpy views of pinned memory
by a thread pool, so a checkpoint loads at host-memory speed.

`export_safetensors` writes a HostWeights blob back out under HF names
(round trip; also how the random-init models can be saved).
"""

from __future__ import annotations

import json
import os
import struct
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

import numpy as np

from ..planning.faults import FormatError, SpecError
from ..planning.graph import ModelSpec, model_from_dict
from .model import Arch, LLAMA3_SCALING, WeightLayout

_ITEMSIZE = {"BF16": 2, "F16": 2, "F32": 4}


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """float16 / float32 array -> bf16 bit patterns (uint16), round to nearest even."""
    f = np.ascontiguousarray(a, dtype=np.float32)
    u = f.view(np.uint32)
    rounded = ((u + (((u >> 16) & 1) + 0x7FFF)) >> 16).astype(np.uint16)
    nan = np.isnan(f)
    if nan.any():
        rounded[nan] = ((u[nan] >> 16) | 0x40).astype(np.uint16)   # keep NaN quiet
    return rounded


class SafetensorsFile:
    """Header + memory map of one .safetensors file."""

    def __init__(self, path: str | os.PathLike):
        self.path = str(path)
        with open(self.path, "rb") as fh:
            head = fh.read(8)
            if len(head) != 8:
                raise FormatError(f"{self.path}: not a safetensors file")
            (n,) = struct.unpack("<Q", head)
            if n > 100 << 20:
                raise FormatError(f"{self.path}: header of {n} bytes")
            doc = json.loads(fh.read(n))
        self.data_start = 8 + n
        self.metadata = doc.pop("__metadata__", {})
        self.entries = doc
        self._mm = np.memmap(self.path, dtype=np.uint8, mode="r")

    def raw(self, name: str) -> tuple[str, tuple, np.ndarray]:
        e = self.entries[name]
        dtype = e["dtype"]
        if dtype not in _ITEMSIZE:
            raise FormatError(f"{self.path}: tensor {name} has unsupported dtype {dtype}")
        b0, b1 = e["data_offsets"]
        shape = tuple(e["shape"])
        want = int(np.prod(shape, dtype=np.int64)) * _ITEMSIZE[dtype]
        if b1 - b0 != want:
            raise FormatError(f"{self.path}: tensor {name} spans {b1 - b0} bytes, shape needs {want}")
        return dtype, shape, self._mm[self.data_start + b0:self.data_start + b1]


class Checkpoint:
    """A directory with config.json and safetensors shard(s), or explicit files."""

    def __init__(self, path: str | os.PathLike, files: list | None = None):
        p = Path(path)
        self.dir = p if p.is_dir() else p.parent
        self.config = {}
        if (self.dir / "config.json").exists():
            self.config = json.loads((self.dir / "config.json").read_text())
        if files is None:
            if p.is_file():
                files = [p]
            else:
                index = self.dir / "model.safetensors.index.json"
                if index.exists():
                    wm = json.loads(index.read_text())["weight_map"]
                    files = sorted({self.dir / f for f in wm.values()})
                else:
                    files = sorted(self.dir.glob("*.safetensors"))
        if not files:
            raise FormatError(f"{path}: no safetensors files")
        self.files = [SafetensorsFile(f) for f in files]
        self.where: dict[str, SafetensorsFile] = {}
        for f in self.files:
            for name in f.entries:
                self.where[name] = f

    def has(self, name: str) -> bool:
        return name in self.where

    def bf16(self, name: str, shape: tuple) -> np.ndarray:
        """Tensor `name` as bf16 bits (uint16) of the given 2-D shape."""
        f = self.where.get(name)
        if f is None:
            raise FormatError(f"checkpoint has no tensor {name}")
        dtype, src_shape, raw = f.raw(name)
        n = int(np.prod(shape, dtype=np.int64))
        if int(np.prod(src_shape, dtype=np.int64)) != n:
            raise FormatError(f"{name}: shape {src_shape} does not fit {shape}")
        if dtype == "BF16":
            return raw.view(np.uint16).reshape(shape)
        src = raw.view(np.float16 if dtype == "F16" else np.float32)
        return bf16_bits(src).reshape(shape)


def open_checkpoint(path: str | os.PathLike):
    """A `.gguf` file (runtime/gguf.py) or a safetensors directory / file."""
    if str(path).endswith(".gguf"):
        from .gguf import GgufCheckpoint
        return GgufCheckpoint(path)
    return Checkpoint(path)


# -- config.json -> (ModelSpec, Arch) -----------------------------------------------

SUPPORTED_ARCHS = frozenset({"LlamaForCausalLM", "Qwen3ForCausalLM", "Qwen3MoeForCausalLM"})
SUPPORTED_MODEL_TYPES = frozenset({"llama", "qwen3", "qwen3_moe"})

def spec_from_hf_config(cfg: dict, name: str | None = None, max_context: int | None = None,
                        seed: int = 0) -> tuple[ModelSpec, Arch]:
    """Llama / Qwen3 / Qwen3-MoE config.json -> the planner's ModelSpec (bf16
    everywhere) and the numerics the spec does not carry."""
    arch_name = (cfg.get("architectures") or [""])[0]
    model_type = cfg.get("model_type", "")
    if arch_name not in SUPPORTED_ARCHS and model_type not in SUPPORTED_MODEL_TYPES:
        raise SpecError(f"unsupported architecture {arch_name or '?'} / model_type {model_type or '?'}: "
                        f"this build executes {sorted(SUPPORTED_ARCHS)}")
    for key, bad in (("attention_bias", True), ("mlp_bias", True)):
        if cfg.get(key) == bad:
            raise SpecError(f"config sets {key}={bad}: biased projections are not implemented")
    act = cfg.get("hidden_act", "silu")
    if act != "silu":
        raise SpecError(f"hidden_act {act!r} is not implemented (SwiGLU with silu only)")
    if cfg.get("use_sliding_window"):
        raise SpecError("sliding-window attention is not implemented")
    if cfg.get("mlp_only_layers"):
        raise SpecError("mlp_only_layers (dense layers inside a MoE model) are not implemented")
    if cfg.get("num_experts") and cfg.get("decoder_sparse_step", 1) != 1:
        raise SpecError("decoder_sparse_step != 1 (dense layers inside a MoE model) is not implemented")
    d = cfg["hidden_size"]
    heads = cfg["num_attention_heads"]
    moe = None
    if cfg.get("num_experts"):
        moe = {"n_experts": cfg["num_experts"], "top_k": cfg["num_experts_per_tok"],
               "expert_ffn_dim": cfg["moe_intermediate_size"]}
        if not cfg.get("norm_topk_prob", True):
            raise SpecError("only norm_topk_prob=true MoE routing is implemented")
    doc = {"format": "model-spec/v1", "name": name or cfg.get("_name_or_path") or arch_name or "hf-model",
           "n_layers": cfg["num_hidden_layers"], "d_model": d, "n_heads": heads,
           "n_kv_heads": cfg.get("num_key_value_heads", heads),
           "head_dim": cfg.get("head_dim") or d // heads, "ffn_dim": cfg["intermediate_size"],
           "vocab_size": cfg["vocab_size"],
           "max_context": max_context or cfg.get("max_position_embeddings", 4096),
           "quant": {"activations": 2.0, "attn_weights": 2.0, "ffn_weights": 2.0, "kv_cache": 2.0,
                     "output_weights": 2.0},
           "gated_ffn": True, "elementwise_epsilon": 0.02, "moe": moe}
    spec = model_from_dict(doc)
    rs = cfg.get("rope_scaling")
    scaling = None
    if rs:
        kind = rs.get("rope_type", rs.get("type"))
        if kind != "llama3":
            raise SpecError(f"rope_scaling type {kind!r} is not implemented")
        scaling = {k: float(rs.get(k, LLAMA3_SCALING[k])) for k in LLAMA3_SCALING}
    qk_norm = "Qwen3" in arch_name or cfg.get("model_type", "").startswith("qwen3")
    arch = Arch(rope_theta=float(cfg.get("rope_theta", 10000.0)), rope_scaling=scaling, qk_norm=qk_norm,
                rms_eps=float(cfg.get("rms_norm_eps", 1e-5)), seed=seed)
    return spec, arch


# -- HF tensor names of the executor's logical tensors --------------------------------

def hf_name(logical: str, tied: bool = False) -> str:
    if logical == "embed":
        return "model.embed_tokens.weight"
    if logical == "final_norm":
        return "model.norm.weight"
    if logical == "lm_head":
        return "model.embed_tokens.weight" if tied else "lm_head.weight"
    layer, rest = logical.split(".", 1)
    i = int(layer[1:])
    p = f"model.layers.{i}."
    simple = {"attn_norm": "input_layernorm.weight", "ffn_norm": "post_attention_layernorm.weight",
              "wq": "self_attn.q_proj.weight", "wk": "self_attn.k_proj.weight",
              "wv": "self_attn.v_proj.weight", "wo": "self_attn.o_proj.weight",
              "q_norm": "self_attn.q_norm.weight", "k_norm": "self_attn.k_norm.weight",
              "w_gate": "mlp.gate_proj.weight", "w_up": "mlp.up_proj.weight",
              "w_down": "mlp.down_proj.weight", "router": "mlp.gate.weight"}
    if rest in simple:
        return p + simple[rest]
    e, w = rest.split(".", 1)                 # e{e}.w_gate / w_up / w_down
    proj = {"w_gate": "gate_proj", "w_up": "up_proj", "w_down": "down_proj"}[w]
    return p + f"mlp.experts.{int(e[1:])}.{proj}.weight"


def _copy_jobs(layout: WeightLayout, tied: bool):
    """(logical tensor, destination byte offset in the blob, rows, cols, mode) for
    every source tensor; mode is 'plain', or ('il', parity) for interleaved rows."""
    for blob in layout.blobs.values():
        for t in blob.tensors.values():
            dst = blob.offset + t.offset
            kind = t.init[0]
            if kind == "plain":
                yield t.init[1], dst, t.rows, t.cols, "plain"
            elif kind == "concat":
                for name, rows in t.init[1]:
                    yield name, dst, rows, t.cols, "plain"
                    dst += rows * t.cols * 2
            elif kind == "interleaved":
                yield t.init[1], dst, t.rows // 2, t.cols, ("il", 0)
                yield t.init[2], dst, t.rows // 2, t.cols, ("il", 1)


def fill_from_checkpoint(layout: WeightLayout, blob: np.ndarray, embed: np.ndarray, ckpt: Checkpoint,
                         threads: int = 8) -> int:
    """Fill the host blob (uint8 [total_bytes]) and embedding table (uint8
    [embed_bytes]) from `ckpt`; returns the bytes written."""
    spec = layout.spec
    tied = not ckpt.has("lm_head.weight") and ckpt.has("model.embed_tokens.weight")
    jobs = list(_copy_jobs(layout, tied))

    def run(job):
        logical, dst, rows, cols, mode = job
        src = ckpt.bf16(hf_name(logical, tied), (rows, cols))
        if mode == "plain":
            blob[dst:dst + rows * cols * 2].view(np.uint16).reshape(rows, cols)[:] = src
        else:
            parity = mode[1]
            full = blob[dst:dst + 2 * rows * cols * 2].view(np.uint16).reshape(2 * rows, cols)
            full[parity::2] = src
        return rows * cols * 2

    consumed = {hf_name(j[0], tied) for j in jobs} | {"model.embed_tokens.weight"}
    names = getattr(ckpt, "where", None)
    if names is not None:
        # every weight the checkpoint carries must be one the layout executes: a tensor
        # left over (biases, extra norms, another architecture's blocks) would be
        # silently ignored and the outputs would be wrong
        extra = sorted(n for n in names if n not in consumed and not n.endswith("rotary_emb.inv_freq"))
        if extra:
            raise FormatError(f"checkpoint tensors this layout does not consume: {extra[:8]}"
                              f"{' ...' if len(extra) > 8 else ''} ({len(extra)} total)")
    with ThreadPoolExecutor(max_workers=threads) as pool:
        total = sum(pool.map(run, jobs))
    e = ckpt.bf16("model.embed_tokens.weight", (spec.vocab_size, spec.d_model))
    embed.view(np.uint16).reshape(spec.vocab_size, spec.d_model)[:] = e
    return total + e.nbytes


# -- writing ---------------------------------------------------------------------------

def write_safetensors(path: str | os.PathLike, tensors: dict, metadata: dict | None = None) -> None:
    """tensors: name -> (dtype 'BF16'|'F16'|'F32', shape, bytes-like)."""
    header, off = {}, 0
    for name, (dtype, shape, data) in tensors.items():
        n = len(memoryview(data).cast("B"))
        header[name] = {"dtype": dtype, "shape": list(shape), "data_offsets": [off, off + n]}
        off += n
    if metadata:
        header["__metadata__"] = {k: str(v) for k, v in metadata.items()}
    blob = json.dumps(header, separators=(",", ":")).encode()
    blob += b" " * (-len(blob) % 8)
    with open(path, "wb") as fh:
        fh.write(struct.pack("<Q", len(blob)))
        fh.write(blob)
        for _, (_, _, data) in tensors.items():
            fh.write(memoryview(data).cast("B"))


def hf_config(spec: ModelSpec, arch: Arch) -> dict:
    """config.json for `spec` (Llama or Qwen3-MoE flavoured)."""
    cfg = {"architectures": ["Qwen3MoeForCausalLM" if spec.moe else
                             ("Qwen3ForCausalLM" if arch.qk_norm else "LlamaForCausalLM")],
           "model_type": "qwen3_moe" if spec.moe else ("qwen3" if arch.qk_norm else "llama"),
           "hidden_size": spec.d_model, "num_hidden_layers": spec.n_layers,
           "num_attention_heads": spec.n_heads, "num_key_value_heads": spec.n_kv_heads,
           "head_dim": spec.head_dim, "intermediate_size": spec.ffn_dim, "vocab_size": spec.vocab_size,
           "max_position_embeddings": spec.max_context, "rms_norm_eps": arch.rms_eps,
           "rope_theta": arch.rope_theta, "tie_word_embeddings": False, "torch_dtype": "bfloat16",
           "_name_or_path": spec.name}
    if arch.rope_scaling:
        cfg["rope_scaling"] = dict(arch.rope_scaling, rope_type="llama3")
    if spec.moe:
        cfg.update(num_experts=spec.moe.n_experts, num_experts_per_tok=spec.moe.top_k,
                   moe_intermediate_size=spec.moe.expert_ffn_dim, norm_topk_prob=True)
    return cfg


def export_safetensors(layout: WeightLayout, blob: np.ndarray, embed: np.ndarray, out_dir: str | os.PathLike,
                       max_shard_bytes: int = 4 << 30) -> list:
    """Write config.json + HF-named bf16 safetensors shard(s) from a filled blob."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    spec = layout.spec
    items = [("model.embed_tokens.weight", (spec.vocab_size, spec.d_model), embed.view(np.uint16))]
    for logical, dst, rows, cols, mode in _copy_jobs(layout, False):
        if mode == "plain":
            a = blob[dst:dst + rows * cols * 2].view(np.uint16).reshape(rows, cols)
        else:
            full = blob[dst:dst + 2 * rows * cols * 2].view(np.uint16).reshape(2 * rows, cols)
            a = np.ascontiguousarray(full[mode[1]::2])
        shape = (cols,) if rows == 1 else (rows, cols)
        items.append((hf_name(logical), shape, a))
    files, cur, size, weight_map = [], {}, 0, {}

    def flush():
        nonlocal cur, size
        if cur:
            name = f"model-{len(files) + 1:05d}.safetensors"
            write_safetensors(out / name, cur, {"format": "pt"})
            for k in cur:
                weight_map[k] = name
            files.append(out / name)
            cur, size = {}, 0

    for name, shape, a in items:
        if size and size + a.nbytes > max_shard_bytes:
            flush()
        cur[name] = ("BF16", shape, np.ascontiguousarray(a))
        size += a.nbytes
    flush()
    (out / "model.safetensors.index.json").write_text(json.dumps(
        {"metadata": {"total_size": int(sum(a.nbytes for _, _, a in items))}, "weight_map": weight_map},
        indent=1))
    (out / "config.json").write_text(json.dumps(hf_config(spec, layout.arch), indent=1))
    return files
