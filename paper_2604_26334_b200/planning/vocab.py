"""Op vocabulary shared by the shard graph, the cost database and the planner.

Restates `pkg/src/shardplan/kernels.py:17-103`: op kinds, the two execution
backends, the contention states a CPU benchmark is taken under, the five
quantization classes (bytes per element) and the canonical FLOP / byte
accounting of a benchmark grid point. Every arithmetic expression keeps the
reference's evaluation order because plan parity is checked bit for bit.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from enum import Enum

__all__ = ["OpKind", "Backend", "Contention", "QUANT_CLASSES", "quant_class_for",
           "KernelRequest", "canonical_workload", "matmul_flops"]


class OpKind(Enum):
    MATMUL = "matmul"
    GQA = "gqa"
    MHA = "mha"
    MOE_ROUTE = "moe_route"
    ELEMENT_WISE = "element_wise"


class Backend(Enum):
    CPU = "cpu"
    GPU = "gpu"


class Contention(Enum):
    STANDALONE = "standalone"
    UNDER_PCIE_TRAFFIC = "under_pcie_traffic"


# Insertion order matters: the install-phase grid iterates classes in this
# order (`kernels.py:38-44`), and the profile file order follows from it.
QUANT_CLASSES: dict[str, float] = {
    "f32": 4.0,
    "f16": 2.0,
    "q8": 1.0,
    "q4": 0.5625,
    "q2": 0.3203125,
}

# Classes by ascending width; `min` keeps the first of equal distances.
_BY_WIDTH = tuple(sorted(QUANT_CLASSES.items(), key=lambda item: item[1]))


def quant_class_for(bytes_per_elem: float) -> str:
    """Nearest benchmarked class to an arbitrary width, measured in log space
    (`kernels.py:50-54`)."""
    if bytes_per_elem <= 0:
        raise ValueError(f"bytes_per_elem must be positive, got {bytes_per_elem}")
    want = math.log(bytes_per_elem)
    best_name, best_gap = None, None
    for name, width in _BY_WIDTH:
        gap = abs(math.log(width) - want)
        if best_gap is None or gap < best_gap:
            best_name, best_gap = name, gap
    return best_name


@dataclass(frozen=True)
class KernelRequest:
    """A priced kernel invocation: (op, quant class, dims, flops, bytes)."""

    op_kind: OpKind
    quant_class: str
    dims: tuple[int, ...]
    flops: float
    bytes: float


_ACT_BPE = 2.0  # activations are benchmarked at f16 width


def _matmul_work(dims, bpe):
    m, k, n = dims
    return 2.0 * m * k * n, k * n * bpe + m * k * _ACT_BPE + m * n * _ACT_BPE


def _attention_work(dims, bpe):
    # GQA dims (t, ctx, h, kv, hd); MHA dims (t, ctx, h, hd). Cache traffic is
    # priced by the KV shard's element-wise kernel, not here.
    t, ctx, heads, head_dim = dims[0], dims[1], dims[2], dims[-1]
    return 4.0 * t * ctx * heads * head_dim, 2.0 * t * heads * head_dim * _ACT_BPE


def _route_work(dims, bpe):
    t, d_model, n_experts = dims
    return (2.0 * t * d_model * n_experts,
            d_model * n_experts * bpe + t * (d_model + n_experts) * _ACT_BPE)


def _elementwise_work(dims, bpe):
    (n,) = dims
    return float(n), n * bpe


_WORK = {
    OpKind.MATMUL: _matmul_work,
    OpKind.GQA: _attention_work,
    OpKind.MHA: _attention_work,
    OpKind.MOE_ROUTE: _route_work,
    OpKind.ELEMENT_WISE: _elementwise_work,
}


def canonical_workload(op_kind: OpKind, dims: tuple[int, ...], bpe: float) -> tuple[float, float]:
    """(flops, bytes) of the benchmark kernel at one grid point
    (`kernels.py:68-98`)."""
    fn = _WORK.get(op_kind)
    if fn is None:
        raise ValueError(f"unknown op kind {op_kind}")
    if op_kind is OpKind.GQA and len(dims) != 5:
        raise ValueError("GQA dims are (t, ctx, heads, kv_heads, head_dim)")
    if op_kind is OpKind.MHA and len(dims) != 4:
        raise ValueError("MHA dims are (t, ctx, heads, head_dim)")
    return fn(dims, bpe)


def matmul_flops(m: int, n: int, k: int) -> int:
    """2 flops per multiply-accumulate of an (m x k) @ (k x n) product."""
    return 2 * m * n * k
