"""Sub-layer shard graph of a decoder-only transformer.

Restates `pkg/src/shardplan/model_graph.py:33-414`. A model is cut into
`3 * n_layers + 1` shards in topological order — per layer an attention
shard, a KV-cache shard and an FFN (or MoE expert-group) shard, then the
output head — each with a fixed priority (attention 0 < KV 1 < FFN/MoE 2 <
head 3) that drives pinning. Each shard prices one pass analytically as a
list of kernel requests.

Arithmetic keeps the reference's association order everywhere (plans are
compared byte for byte after `repr`). Embedding tables and RMSNorm vectors
are not shards in the reference and are not shards here; the executor
handles them by policy ("Memory outside the plan").
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from enum import Enum
from pathlib import Path

from .faults import FormatError, SpecError
from .vocab import KernelRequest, OpKind, quant_class_for

__all__ = ["MODEL_FORMAT", "TENSOR_CLASSES", "HEAD_ROWS_CAP", "DEFAULT_ELEMENTWISE_EPSILON",
           "ShardKind", "PRIORITY", "MoeSpec", "ModelSpec", "ShardCost", "SubLayerShard",
           "shard_cost", "kv_cache_bytes", "total_model_bytes", "build_shards",
           "model_to_dict", "model_from_dict", "load_model", "save_model",
           "attention_weight_bytes", "ffn_weight_bytes", "head_weight_bytes"]

MODEL_FORMAT = "model-spec/v1"
TENSOR_CLASSES = ("attn_weights", "ffn_weights", "output_weights", "kv_cache", "activations")

# Only sampled positions produce logits: at most 64 rows per pass
# (`model_graph.py:30-33`).
HEAD_ROWS_CAP = 64
DEFAULT_ELEMENTWISE_EPSILON = 0.02


class ShardKind(Enum):
    ATTENTION = "attention"
    KV_CACHE = "kv_cache"
    FFN = "ffn"
    MOE_EXPERT_GROUP = "moe_expert_group"
    OUTPUT_HEAD = "output_head"


PRIORITY: dict[ShardKind, int] = {
    ShardKind.ATTENTION: 0,
    ShardKind.KV_CACHE: 1,
    ShardKind.FFN: 2,
    ShardKind.MOE_EXPERT_GROUP: 2,
    ShardKind.OUTPUT_HEAD: 3,
}


@dataclass(frozen=True)
class MoeSpec:
    n_experts: int
    top_k: int
    expert_ffn_dim: int


@dataclass(frozen=True)
class ModelSpec:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    ffn_dim: int
    vocab_size: int
    max_context: int
    quant: dict[str, float]     # tensor class -> bytes per element
    moe: MoeSpec | None = None
    gated_ffn: bool = True
    elementwise_epsilon: float = DEFAULT_ELEMENTWISE_EPSILON

    def __post_init__(self):
        for field in ("n_layers", "d_model", "n_heads", "n_kv_heads", "head_dim",
                      "ffn_dim", "vocab_size", "max_context"):
            value = getattr(self, field)
            if value <= 0:
                raise SpecError(f"{self.name}: {field} must be positive, got {value}")
        if self.n_heads % self.n_kv_heads:
            raise SpecError(
                f"{self.name}: n_heads ({self.n_heads}) must be a multiple of "
                f"n_kv_heads ({self.n_kv_heads})")
        absent = [c for c in TENSOR_CLASSES if c not in self.quant]
        if absent:
            raise SpecError(f"{self.name}: quant map missing classes {absent}")
        for cls, bpe in self.quant.items():
            if bpe <= 0:
                raise SpecError(f"{self.name}: quant[{cls}] must be positive, got {bpe}")
        moe = self.moe
        if moe is not None:
            if min(moe.n_experts, moe.top_k, moe.expert_ffn_dim) <= 0:
                raise SpecError(f"{self.name}: moe counts must be positive")
            if moe.top_k > moe.n_experts:
                raise SpecError(f"{self.name}: moe top_k exceeds n_experts")
        if not (0 <= self.elementwise_epsilon < 1):
            raise SpecError(f"{self.name}: elementwise_epsilon must be in [0, 1)")

    @property
    def ffn_mats(self) -> int:
        """Weight matrices per FFN: gate, up, down when gated; else up, down."""
        return 3 if self.gated_ffn else 2

    def activation_bytes(self, new_tokens: int) -> float:
        """One hidden-state tensor passed between shards (`model_graph.py:112-114`)."""
        return new_tokens * self.d_model * self.quant["activations"]


@dataclass(frozen=True)
class ShardCost:
    flops: float
    read_bytes: float
    write_bytes: float


# -- per-kind pricing (`model_graph.py:137-211`) -------------------------------

def _price_attention(shard, t, ctx, eps, qa):
    s = shard.spec
    width = 4 * s.n_heads * s.head_dim
    proj = KernelRequest(
        OpKind.MATMUL, quant_class_for(s.quant["attn_weights"]), (t, s.d_model, width),
        flops=2.0 * t * s.d_model * width * eps,
        bytes=shard.weight_bytes + t * s.d_model * qa + t * width * qa)
    if s.n_kv_heads == s.n_heads:
        op, dims = OpKind.MHA, (t, ctx, s.n_heads, s.head_dim)
    else:
        op, dims = OpKind.GQA, (t, ctx, s.n_heads, s.n_kv_heads, s.head_dim)
    core = KernelRequest(
        op, quant_class_for(s.quant["kv_cache"]), dims,
        flops=4.0 * t * ctx * s.n_heads * s.head_dim * eps,
        bytes=2.0 * t * s.n_heads * s.head_dim * qa)
    return [proj, core]


def _price_kv(shard, t, ctx, eps, qa):
    s = shard.spec
    qkv = s.quant["kv_cache"]
    # every resident request cache is touched once, plus the appended rows
    elems = 2 * (shard.kv_replicas * ctx + t) * s.n_kv_heads * s.head_dim
    return [KernelRequest(OpKind.ELEMENT_WISE, quant_class_for(qkv), (elems,),
                          flops=float(elems), bytes=elems * qkv)]


def _price_ffn(shard, t, ctx, eps, qa):
    s = shard.spec
    width = s.ffn_mats * s.ffn_dim
    return [KernelRequest(
        OpKind.MATMUL, quant_class_for(s.quant["ffn_weights"]), (t, s.d_model, width),
        flops=2.0 * t * s.d_model * width * eps,
        bytes=shard.weight_bytes + 2.0 * t * (s.d_model + s.ffn_dim) * qa)]


def _price_moe(shard, t, ctx, eps, qa):
    s = shard.spec
    moe = s.moe
    qf = s.quant["ffn_weights"]
    cls = quant_class_for(qf)
    router = KernelRequest(
        OpKind.MOE_ROUTE, cls, (t, s.d_model, moe.n_experts),
        flops=2.0 * t * s.d_model * moe.n_experts * eps,
        bytes=s.d_model * moe.n_experts * qf + t * (s.d_model + moe.n_experts) * qa)
    touched = min(moe.n_experts, t * moe.top_k)
    per_expert = s.ffn_mats * s.d_model * moe.expert_ffn_dim * qf
    width = s.ffn_mats * moe.expert_ffn_dim
    experts = KernelRequest(
        OpKind.MATMUL, cls, (t * moe.top_k, s.d_model, width),
        flops=2.0 * t * moe.top_k * s.d_model * width * eps,
        bytes=(touched * per_expert
               + t * moe.top_k * (s.d_model + 2 * moe.expert_ffn_dim) * qa
               + t * s.d_model * qa))
    return [router, experts]


def _price_head(shard, t, ctx, eps, qa):
    s = shard.spec
    rows = min(t, HEAD_ROWS_CAP)
    return [KernelRequest(
        OpKind.MATMUL, quant_class_for(s.quant["output_weights"]),
        (rows, s.d_model, s.vocab_size),
        flops=2.0 * rows * s.d_model * s.vocab_size * eps,
        bytes=shard.weight_bytes + rows * (s.d_model + s.vocab_size) * qa)]


_PRICERS = {
    ShardKind.ATTENTION: _price_attention,
    ShardKind.KV_CACHE: _price_kv,
    ShardKind.FFN: _price_ffn,
    ShardKind.MOE_EXPERT_GROUP: _price_moe,
    ShardKind.OUTPUT_HEAD: _price_head,
}


@dataclass(frozen=True)
class SubLayerShard:
    """One schedulable unit of the decoder: footprint + pure cost functions."""

    id: int
    layer_index: int
    kind: ShardKind
    weight_bytes: float
    priority: int
    spec: ModelSpec
    context_len: int
    kv_replicas: int = 1

    def kernels(self, new_tokens: int, context_len: int) -> list[KernelRequest]:
        if new_tokens < 1:
            raise SpecError(f"new_tokens must be >= 1, got {new_tokens}")
        pricer = _PRICERS.get(self.kind)
        if pricer is None:
            raise SpecError(f"unhandled shard kind {self.kind}")
        s = self.spec
        return pricer(self, new_tokens, context_len, 1.0 + s.elementwise_epsilon,
                      s.quant["activations"])

    def cost(self, new_tokens: int, context_len: int) -> ShardCost:
        return shard_cost(self, new_tokens, context_len)

    def peak_activation_bytes(self, new_tokens: int) -> float:
        """Live activation working set of one pass (`model_graph.py:216-239`)."""
        s = self.spec
        qa = s.quant["activations"]
        t = new_tokens
        kind = self.kind
        if kind is ShardKind.ATTENTION:
            return t * (s.d_model + 4 * s.n_heads * s.head_dim) * qa
        if kind is ShardKind.KV_CACHE:
            return 0.0
        if kind is ShardKind.FFN:
            inner = 2 * s.ffn_dim if s.gated_ffn else s.ffn_dim
            return t * (s.d_model + inner) * qa
        if kind is ShardKind.MOE_EXPERT_GROUP:
            moe = s.moe
            inner = 2 * moe.expert_ffn_dim if s.gated_ffn else moe.expert_ffn_dim
            return t * (s.d_model + inner) * qa + t * moe.n_experts * qa
        if kind is ShardKind.OUTPUT_HEAD:
            return min(t, HEAD_ROWS_CAP) * (s.d_model + s.vocab_size) * qa
        raise SpecError(f"unhandled shard kind {kind}")

    def kv_append_bytes(self, new_tokens: int) -> float:
        """Cache bytes appended per pass; 0 for non-KV shards (`:241-246`)."""
        if self.kind is not ShardKind.KV_CACHE:
            return 0.0
        s = self.spec
        return 2.0 * new_tokens * s.n_kv_heads * s.head_dim * s.quant["kv_cache"]


def shard_cost(shard: SubLayerShard, new_tokens: int, context_len: int) -> ShardCost:
    """Sum of a shard's kernels split into reads and writes (`:249-276`)."""
    if new_tokens < 1:
        raise SpecError(f"new_tokens must be >= 1, got {new_tokens}")
    s = shard.spec
    qa = s.quant["activations"]
    t = new_tokens
    reqs = shard.kernels(new_tokens, context_len)
    flops = sum(r.flops for r in reqs)
    moved = sum(r.bytes for r in reqs)
    kind = shard.kind
    if kind is ShardKind.ATTENTION:
        written = t * (4 * s.n_heads * s.head_dim + s.n_heads * s.head_dim) * qa
    elif kind is ShardKind.KV_CACHE:
        written = shard.kv_append_bytes(t)
    elif kind is ShardKind.FFN:
        written = t * (s.d_model + s.ffn_dim) * qa
    elif kind is ShardKind.MOE_EXPERT_GROUP:
        moe = s.moe
        written = t * moe.n_experts * qa + t * (moe.top_k * moe.expert_ffn_dim + s.d_model) * qa
    else:
        written = min(t, HEAD_ROWS_CAP) * s.vocab_size * qa
    return ShardCost(flops=flops, read_bytes=moved - written, write_bytes=written)


# -- footprints (`model_graph.py:279-310`) -------------------------------------

def attention_weight_bytes(s: ModelSpec) -> float:
    """Q, O (d x h*hd each) and K, V (d x kv*hd each)."""
    count = 2 * s.d_model * s.n_heads * s.head_dim + 2 * s.d_model * s.n_kv_heads * s.head_dim
    return count * s.quant["attn_weights"]


def ffn_weight_bytes(s: ModelSpec) -> float:
    qf = s.quant["ffn_weights"]
    if s.moe is None:
        return s.ffn_mats * s.d_model * s.ffn_dim * qf
    count = (s.moe.n_experts * s.ffn_mats * s.d_model * s.moe.expert_ffn_dim
             + s.d_model * s.moe.n_experts)
    return count * qf


def head_weight_bytes(s: ModelSpec) -> float:
    return s.d_model * s.vocab_size * s.quant["output_weights"]


def kv_cache_bytes(spec: ModelSpec, context_len: int) -> float:
    """All layers' K and V for one request at `context_len` positions."""
    if context_len < 0:
        raise SpecError(f"context_len must be >= 0, got {context_len}")
    return (2.0 * spec.n_layers * spec.n_kv_heads * spec.head_dim
            * context_len * spec.quant["kv_cache"])


def total_model_bytes(spec: ModelSpec) -> float:
    per_layer = attention_weight_bytes(spec) + ffn_weight_bytes(spec)
    return spec.n_layers * per_layer + head_weight_bytes(spec)


def build_shards(spec: ModelSpec, context_len: int, kv_replicas: int = 1) -> list[SubLayerShard]:
    """Shards in topological order: [Attn_i, KV_i, FFN_i|MoE_i] * L + head."""
    if context_len < 0:
        raise SpecError(f"context_len must be >= 0, got {context_len}")
    if context_len > spec.max_context:
        raise SpecError(
            f"{spec.name}: context_len {context_len} exceeds max_context {spec.max_context}")
    if kv_replicas < 1:
        raise SpecError(f"kv_replicas must be >= 1, got {kv_replicas}")
    ffn_kind = ShardKind.FFN if spec.moe is None else ShardKind.MOE_EXPERT_GROUP
    per_layer = (
        (ShardKind.ATTENTION, attention_weight_bytes(spec)),
        (ShardKind.KV_CACHE, kv_replicas * kv_cache_bytes(spec, context_len) / spec.n_layers),
        (ffn_kind, ffn_weight_bytes(spec)),
    )
    layout = [(layer, kind, w) for layer in range(spec.n_layers) for kind, w in per_layer]
    layout.append((spec.n_layers, ShardKind.OUTPUT_HEAD, head_weight_bytes(spec)))
    return [SubLayerShard(id=i, layer_index=layer, kind=kind, weight_bytes=w,
                          priority=PRIORITY[kind], spec=spec, context_len=context_len,
                          kv_replicas=kv_replicas)
            for i, (layer, kind, w) in enumerate(layout)]


# -- model-spec/v1 JSON ----------------------------------------------------------

def model_to_dict(s: ModelSpec) -> dict:
    moe = None
    if s.moe is not None:
        moe = {"n_experts": s.moe.n_experts, "top_k": s.moe.top_k,
               "expert_ffn_dim": s.moe.expert_ffn_dim}
    return {
        "format": MODEL_FORMAT, "name": s.name, "n_layers": s.n_layers,
        "d_model": s.d_model, "n_heads": s.n_heads, "n_kv_heads": s.n_kv_heads,
        "head_dim": s.head_dim, "ffn_dim": s.ffn_dim, "vocab_size": s.vocab_size,
        "max_context": s.max_context, "quant": dict(s.quant), "gated_ffn": s.gated_ffn,
        "elementwise_epsilon": s.elementwise_epsilon, "moe": moe,
    }


def model_from_dict(doc: dict) -> ModelSpec:
    if doc.get("format") != MODEL_FORMAT:
        raise FormatError(f"expected {MODEL_FORMAT}, got {doc.get('format')!r}")
    moe_doc = doc.get("moe")
    moe = None
    if moe_doc:
        moe = MoeSpec(n_experts=int(moe_doc["n_experts"]), top_k=int(moe_doc["top_k"]),
                      expert_ffn_dim=int(moe_doc["expert_ffn_dim"]))
    ints = {f: int(doc[f]) for f in ("n_layers", "d_model", "n_heads", "n_kv_heads",
                                      "head_dim", "ffn_dim", "vocab_size", "max_context")}
    return ModelSpec(
        name=doc["name"], quant={k: float(v) for k, v in doc["quant"].items()}, moe=moe,
        gated_ffn=bool(doc.get("gated_ffn", True)),
        elementwise_epsilon=float(doc.get("elementwise_epsilon", DEFAULT_ELEMENTWISE_EPSILON)),
        **ints)


def load_model(path: str | Path) -> ModelSpec:
    return model_from_dict(json.loads(Path(path).read_text(encoding="utf-8")))


def save_model(s: ModelSpec, path: str | Path) -> None:
    Path(path).write_text(json.dumps(model_to_dict(s), indent=2, sort_keys=True) + "\n",
                          encoding="utf-8")
