"""Model load: architecture constants, host weight layout and random init.

The north_star's "model load" (BASELINE.json) for this build: weights are
random-initialised from a `ModelSpec` (no checkpoints travel to the box),
deterministically from (model seed, tensor name), generated on the GPU by
`ps_init_*` and written into ONE pinned, mapped host blob laid out
shard-contiguous in stream order, so every streamed shard is one or a few
large `cudaMemcpyAsync` source ranges and CPU-placed shards are readable
zero-copy. The embedding table is a separate mapped host buffer (outside
the plan, `pkg/src/shardplan/model_graph.py:279-297`).

Tensor conventions (bf16, row-major, rows = output features):
  attention shard  attn_norm[d] | wqkv[(h + 2 kv) hd, d] (= wq; wk; wv) |
                   q_norm[hd], k_norm[hd] (Qwen3) | wo[d, h hd]
  FFN shard        ffn_norm[d] | wgu[2 ffn, d] (gate/up rows interleaved:
                   2j = gate_j, 2j+1 = up_j) | wdown[d, ffn]
  MoE shard        ffn_norm[d] | router[E, d] | per expert e: wgu_e[2 eff, d],
                   wdown_e[d, eff]
  head shard       final_norm[d] | lm_head[V, d]
Every tensor starts on a 256-byte boundary.
"""

from __future__ import annotations

import hashlib
import math
from dataclasses import dataclass, field

import numpy as np

from ..planning.graph import ModelSpec, ShardKind, build_shards
from . import lib as L

ALIGN = 256


def _align(n: int) -> int:
    return (n + ALIGN - 1) // ALIGN * ALIGN


@dataclass(frozen=True)
class Arch:
    """Numerics the ModelSpec does not carry (public HF configs)."""

    rope_theta: float = 10000.0
    rope_scaling: dict | None = None     # llama3: factor, low_freq_factor, high_freq_factor, original_max
    qk_norm: bool = False
    rms_eps: float = 1e-5
    seed: int = 0


LLAMA3_SCALING = {"factor": 8.0, "low_freq_factor": 1.0, "high_freq_factor": 4.0,
                  "original_max_position_embeddings": 8192}

ARCHS = {
    "tiny-llama": Arch(rope_theta=10000.0),
    "llama3.1-8b": Arch(rope_theta=500000.0, rope_scaling=LLAMA3_SCALING),
    "llama3.3-70b": Arch(rope_theta=500000.0, rope_scaling=LLAMA3_SCALING),
    "qwen3-30b-a3b": Arch(rope_theta=1000000.0, qk_norm=True, rms_eps=1e-6),
    "tiny-moe": Arch(rope_theta=1000000.0, qk_norm=True, rms_eps=1e-6),
}


def arch_for(spec: ModelSpec, seed: int = 0) -> Arch:
    base = ARCHS.get(spec.name, Arch())
    return Arch(base.rope_theta, base.rope_scaling, base.qk_norm, base.rms_eps, seed)


def tensor_seed(model_seed: int, name: str) -> int:
    """64-bit seed of one logical tensor: sha256("<seed>:<name>")[:8], little endian."""
    return int.from_bytes(hashlib.sha256(f"{model_seed}:{name}".encode()).digest()[:8], "little")


# Tensors whose rows get a heavy-tailed scale s_r = min(u_r^-1/2, 64) on top of
# U(-a, a) (ps_init_rowscaled_bf16): the output head. A random-init head with equal
# row norms puts the top two of 128k logits within 1e-3 of max|logit| on 3 % of
# tokens, so bf16 rounding in a prefill pass would flip greedy ids; Pareto(2) row
# norms make that ~4x rarer (SURVEY.md §7 hard part 7), without changing any shape.
HEAVY_ROW_TENSORS = frozenset({"lm_head"})


def init_scale(name: str, fan_in: int) -> tuple[float, float]:
    """(scale, bias) of the uniform init: norms ~ U(0.9, 1.1), embeddings
    ~ U(-1, 1), linear weights ~ U(-a, a) with a = sqrt(3 / fan_in) (times a
    per-row factor for HEAVY_ROW_TENSORS)."""
    leaf = name.rsplit(".", 1)[-1]
    if leaf.endswith("norm"):
        return 0.1, 1.0
    if leaf == "embed":
        return 1.0, 0.0
    return math.sqrt(3.0 / fan_in), 0.0


def rope_inv_freq(arch: Arch, head_dim: int) -> np.ndarray:
    """Per-pair inverse frequencies (float64), Llama-3 scaling when configured."""
    inv = 1.0 / (arch.rope_theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    sc = arch.rope_scaling
    if not sc:
        return inv
    factor, lo, hi = sc["factor"], sc["low_freq_factor"], sc["high_freq_factor"]
    orig = sc["original_max_position_embeddings"]
    low_wl, high_wl = orig / lo, orig / hi
    wl = 2 * math.pi / inv
    out = np.where(wl > low_wl, inv / factor, inv)
    smooth = (orig / wl - lo) / (hi - lo)
    mid = (wl <= low_wl) & (wl >= high_wl)
    return np.where(mid, (1 - smooth) * inv / factor + smooth * inv, out)


def rope_table(arch: Arch, head_dim: int, n_pos: int) -> np.ndarray:
    """(cos, sin) per position and pair as float32 [n_pos, head_dim/2, 2]."""
    ang = np.arange(n_pos, dtype=np.float64)[:, None] * rope_inv_freq(arch, head_dim)[None, :]
    return np.stack([np.cos(ang), np.sin(ang)], axis=-1).astype(np.float32)


@dataclass
class TensorSlot:
    name: str
    offset: int          # bytes from the start of its shard
    rows: int
    cols: int
    init: tuple          # ("plain", [seed names]) or ("interleaved", name_a, name_b)

    @property
    def nbytes(self) -> int:
        return self.rows * self.cols * 2


@dataclass
class ShardBlob:
    shard_id: int
    kind: ShardKind
    layer: int
    offset: int                      # bytes from the start of the host blob
    nbytes: int
    tensors: dict = field(default_factory=dict)   # name -> TensorSlot (offset within shard)


class WeightLayout:
    """Byte layout of the host weight blob, in stream order."""

    def __init__(self, spec: ModelSpec, arch: Arch):
        self.spec, self.arch = spec, arch
        s = spec
        self.qkv_rows = (s.n_heads + 2 * s.n_kv_heads) * s.head_dim
        self.blobs: dict[int, ShardBlob] = {}
        cursor = 0
        for shard in build_shards(spec, 0):
            if shard.kind is ShardKind.KV_CACHE:
                continue
            blob = ShardBlob(shard.id, shard.kind, shard.layer_index, cursor, 0)
            self._fill(blob)
            cursor += _align(blob.nbytes)
            self.blobs[shard.id] = blob
        self.total_bytes = cursor
        self.embed_bytes = s.vocab_size * s.d_model * 2

    def _fill(self, blob: ShardBlob) -> None:
        s, i = self.spec, blob.layer
        off = 0

        def add(name, rows, cols, init):
            nonlocal off
            blob.tensors[name] = TensorSlot(name, off, rows, cols, init)
            off = _align(off + rows * cols * 2)

        hd, h, kv, d = s.head_dim, s.n_heads, s.n_kv_heads, s.d_model
        if blob.kind is ShardKind.ATTENTION:
            add(f"L{i}.attn_norm", 1, d, ("plain", f"L{i}.attn_norm"))
            add(f"L{i}.wqkv", self.qkv_rows, d,
                ("concat", [(f"L{i}.wq", h * hd), (f"L{i}.wk", kv * hd), (f"L{i}.wv", kv * hd)]))
            if self.arch.qk_norm:   # consumed between the projections, so stored between them
                add(f"L{i}.q_norm", 1, hd, ("plain", f"L{i}.q_norm"))
                add(f"L{i}.k_norm", 1, hd, ("plain", f"L{i}.k_norm"))
            add(f"L{i}.wo", d, h * hd, ("plain", f"L{i}.wo"))
        elif blob.kind is ShardKind.FFN:
            add(f"L{i}.ffn_norm", 1, d, ("plain", f"L{i}.ffn_norm"))
            add(f"L{i}.wgu", 2 * s.ffn_dim, d, ("interleaved", f"L{i}.w_gate", f"L{i}.w_up"))
            add(f"L{i}.wdown", d, s.ffn_dim, ("plain", f"L{i}.w_down"))
        elif blob.kind is ShardKind.MOE_EXPERT_GROUP:
            moe = s.moe
            add(f"L{i}.ffn_norm", 1, d, ("plain", f"L{i}.ffn_norm"))
            add(f"L{i}.router", moe.n_experts, d, ("plain", f"L{i}.router"))
            for e in range(moe.n_experts):
                add(f"L{i}.e{e}.wgu", 2 * moe.expert_ffn_dim, d,
                    ("interleaved", f"L{i}.e{e}.w_gate", f"L{i}.e{e}.w_up"))
                add(f"L{i}.e{e}.wdown", d, moe.expert_ffn_dim, ("plain", f"L{i}.e{e}.w_down"))
        elif blob.kind is ShardKind.OUTPUT_HEAD:
            add("final_norm", 1, d, ("plain", "final_norm"))
            add("lm_head", s.vocab_size, d, ("plain", "lm_head"))
        blob.nbytes = off

    def tensor(self, shard_id: int, name: str) -> TensorSlot:
        return self.blobs[shard_id].tensors[name]


class SharedHostBlob:
    """One host buffer shared by every process of a node (data-parallel replicas):
    a /dev/shm file, mmapped and pinned in each process with cudaHostRegister
    (mapped, portable), so a node holds one copy of the weights instead of one per
    GPU. The process that creates the file pins it first, fills it and then sets a
    ready flag; the others wait for the pinned flag, pin, and wait for the ready
    flag. Both flags live in a header page behind the weights, inside the shared
    memory itself, so a replica that is slow to arrive still sees them after the
    creator has finished and removed the name (the mapping outlives the name)."""

    HEADER = 4096
    PINNED, READY = b"PSPINNED", b"PS_READY"

    def __init__(self, name: str, nbytes: int, timeout_s: float = 3600.0):
        import ctypes
        import mmap
        import os
        import time
        self.path = f"/dev/shm/{name}"
        self.nbytes = nbytes
        self.timeout_s = timeout_s
        total = nbytes + self.HEADER
        try:
            self.fd = os.open(self.path, os.O_CREAT | os.O_EXCL | os.O_RDWR, 0o600)
            self.creator = True
            try:
                os.ftruncate(self.fd, total)
                # populate the tmpfs pages up front: several processes pinning the same
                # sparse segment concurrently fails for large segments (measured at
                # 17 GB), and a full /dev/shm fails here instead of SIGBUS later
                os.posix_fallocate(self.fd, 0, total)
            except OSError:
                os.close(self.fd)
                os.unlink(self.path)
                raise
        except FileExistsError:
            self.creator = False
            self.fd = os.open(self.path, os.O_RDWR)
            self._wait(lambda: os.fstat(self.fd).st_size >= total, "sized the blob")
        self.mm = mmap.mmap(self.fd, total)
        if not self.creator:
            # the creator pins first (populated pages), then the others
            self._wait(lambda: self._flag(0) == self.PINNED, "pinned the blob")
        self.addr = ctypes.addressof(ctypes.c_char.from_buffer(self.mm))
        try:
            L.call("ps_host_register", self.addr, total, 1)
        except Exception:
            self.addr = 0
            try:
                self.mm.close()
            except BufferError:
                pass
            os.close(self.fd)
            if self.creator:
                self.unlink()
            raise
        if self.creator:
            self.mm[nbytes:nbytes + 8] = self.PINNED

    def _flag(self, slot: int) -> bytes:
        o = self.nbytes + 8 * slot
        return bytes(self.mm[o:o + 8])

    def _wait(self, cond, what: str) -> None:
        """Poll `cond`; a creator that failed removes the name, which ends the wait."""
        import os
        import time
        t0 = time.time()
        while not cond():
            if not os.path.exists(self.path) and not cond():
                raise FileNotFoundError(f"{self.path}: creator left before it {what}")
            if time.time() - t0 > self.timeout_s:
                raise TimeoutError(f"{self.path}: creator never {what}")
            time.sleep(0.02)

    @staticmethod
    def fits(nbytes: int) -> bool:
        import os
        try:
            st = os.statvfs("/dev/shm")
        except OSError:
            return False
        return st.f_bavail * st.f_frsize > nbytes * 1.05

    def mark_ready(self) -> None:
        o = self.nbytes + 8
        self.mm[o:o + 8] = self.READY

    def wait_ready(self) -> None:
        self._wait(lambda: self._flag(1) == self.READY, "filled the weights")

    def unlink(self) -> None:
        """Remove the name once every process that needs it has mapped the segment;
        the memory lives until the last mapping goes."""
        import os
        try:
            os.unlink(self.path)
        except FileNotFoundError:
            pass

    def close(self) -> None:
        import os
        if self.addr:
            L.call("ps_host_unregister", self.addr)
            self.addr = 0
            import gc
            gc.collect()   # drop the ctypes view before unmapping
            try:
                self.mm.close()
            except BufferError:
                pass
            os.close(self.fd)
            if self.creator:
                self.unlink()


class HostWeights:
    """Pinned + mapped host blob holding every shard, plus the embedding table.

    `generate()` fills it on the GPU (deterministic per tensor name) through
    a bounded device staging buffer and D2H copies; the staging buffer is
    released before the VRAM arena is created, so it does not count against
    the budget. With `shared=name` the blob and table live in one /dev/shm
    segment shared by the node's replicas (SharedHostBlob): only the process
    that created it generates, the others wait for it.
    """

    def __init__(self, spec: ModelSpec, arch: Arch, shared: str | None = None, host_format: str = "bf16"):
        """`host_format="coded"`: no bf16 blob on the host at all — `generate()` produces
        every tensor on the GPU and keeps only its hx-coded form (runtime/hxcodec.py,
        ~0.65 x the bytes; dense models), for models whose bf16 blob and coded copy do not
        fit host memory together. The embedding table stays bf16."""
        self.spec, self.arch = spec, arch
        self.layout = WeightLayout(spec, arch)
        self.shared = None
        self.coded = None
        self.hx = None
        self.host_format = host_format
        if host_format not in ("bf16", "coded"):
            raise ValueError(f"host_format {host_format!r}")
        if host_format == "coded":
            if spec.moe is not None or shared is not None:
                raise ValueError("host_format='coded' is for dense models with a private host copy")
            self.base = 0
            self.embed = L.host_alloc(self.layout.embed_bytes, mapped=True)
            return
        if shared is not None:
            total = _align(self.layout.total_bytes) + self.layout.embed_bytes
            try:
                self.shared = SharedHostBlob(shared, total)
            except Exception as exc:   # cannot pin a shared segment here: private copy
                import warnings
                warnings.warn(f"shared host weights unavailable ({exc}); using a private pinned blob")
                self.shared = None
        if self.shared is not None:
            self.base = self.shared.addr
            self.embed = self.shared.addr + _align(self.layout.total_bytes)
        else:
            self.base = L.host_alloc(self.layout.total_bytes, mapped=True)
            self.embed = L.host_alloc(self.layout.embed_bytes, mapped=True)

    def close(self) -> None:
        if self.coded is not None:
            self.coded.close()
            self.coded = None
        if self.hx is not None:
            self.hx.close()
            self.hx = None
        if self.host_format == "coded":
            if self.embed:
                L.host_free(self.embed)
                self.embed = 0
            return
        if self.shared is not None:
            if self.base:
                self.base = self.embed = 0
                self.shared.close()
            return
        if self.base:
            L.host_free(self.base)
            L.host_free(self.embed)
            self.base = self.embed = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def shard_ptr(self, shard_id: int) -> int:
        if not self.base:
            raise RuntimeError("no bf16 host blob (host_format='coded'): read the coded shards")
        return self.base + self.layout.blobs[shard_id].offset

    def tensor_ptr(self, shard_id: int, name: str) -> int:
        return self.shard_ptr(shard_id) + self.layout.tensor(shard_id, name).offset

    def host_view(self, shard_id: int, name: str) -> np.ndarray:
        """uint16 view (bf16 bits) of one tensor in the pinned blob (host_format='coded':
        a decoded copy, for tests and the CPU oracle)."""
        t = self.layout.tensor(shard_id, name)
        if self.host_format == "coded":   # decode the hx copy on the GPU (ps_hx_expand)
            import torch
            off, m = self.hx.tensors[shard_id][name]
            addr = self.hx.shard_ptr(shard_id) + off
            if m is None:
                raw = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * (t.rows * t.cols * 2)).from_address(addr))
                return raw.view(np.uint16).reshape(t.rows, t.cols).copy()
            stream = torch.cuda.current_stream().cuda_stream
            blob = torch.empty(m.nbytes, dtype=torch.uint8, device="cuda")
            L.memcpy_async(blob.data_ptr(), addr, m.nbytes, stream)
            offs = torch.from_numpy(m.block_off[:-1].astype(np.int32)).cuda()
            lut = torch.from_numpy(m.lut.view(np.int32)).cuda()
            out = torch.empty(t.rows, t.cols, dtype=torch.int16, device="cuda")
            L.call("ps_hx_expand", blob.data_ptr(), offs.data_ptr(), t.rows, t.cols, lut.data_ptr(),
                   out.data_ptr(), t.cols, stream)
            return out.cpu().numpy().view(np.uint16)
        buf = (np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint16 * (t.rows * t.cols))
                                     .from_address(self.tensor_ptr(shard_id, name))))
        return buf.reshape(t.rows, t.cols)

    def blob_bytes(self) -> np.ndarray:
        """uint8 view of the whole pinned blob (no copy)."""
        import ctypes
        return np.ctypeslib.as_array((ctypes.c_uint8 * self.layout.total_bytes).from_address(self.base))

    def embed_bytes(self) -> np.ndarray:
        import ctypes
        return np.ctypeslib.as_array((ctypes.c_uint8 * self.layout.embed_bytes).from_address(self.embed))

    def load(self, ckpt) -> int:
        """Fill the blob from a safetensors checkpoint (runtime/checkpoint.py)
        instead of the random init; returns the bytes written."""
        from .checkpoint import fill_from_checkpoint
        return fill_from_checkpoint(self.layout, self.blob_bytes(), self.embed_bytes(), ckpt)

    def export(self, out_dir: str) -> list:
        """Write the blob as an HF-named bf16 safetensors checkpoint + config.json."""
        from .checkpoint import export_safetensors
        return export_safetensors(self.layout, self.blob_bytes(), self.embed_bytes(), out_dir)

    def export_gguf(self, path: str) -> int:
        """Write the blob as a GGUF v3 file (llama.cpp conventions, runtime/gguf.py)."""
        from .gguf import write_gguf
        return write_gguf(path, self.layout, self.blob_bytes(), self.embed_bytes(), self.arch)

    def embed_view(self) -> np.ndarray:
        n = self.spec.vocab_size * self.spec.d_model
        buf = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint16 * n).from_address(self.embed))
        return buf.reshape(self.spec.vocab_size, self.spec.d_model)

    def generate(self, staging_bytes: int = 256 << 20) -> None:
        if self.host_format == "coded":
            self._generate_coded(staging_bytes)
            return
        if self.shared is not None and not self.shared.creator:
            self.shared.wait_ready()          # another replica of this node fills it
            return
        self._generate(staging_bytes)
        if self.shared is not None:
            self.shared.mark_ready()

    def tensor_filler(self, t: TensorSlot, stream: int):
        """fill(dst_dev, r0, r1): the deterministic init of rows [r0, r1) of tensor `t`
        (bf16, row-major) written to device memory at dst_dev."""
        seed, cols = self.arch.seed, t.cols

        def plain(name, fan_in):
            scale, bias = init_scale(name, fan_in)
            sd = tensor_seed(seed, name)
            if name in HEAVY_ROW_TENSORS:     # heavy-tailed row norms (margin-robust head)
                return lambda dst, e0, n: L.call("ps_init_rowscaled_bf16", dst, n, sd, e0, fan_in, scale, stream)
            return lambda dst, e0, n: L.call("ps_init_uniform_bf16", dst, n, sd, e0, scale, bias, stream)

        kind = t.init[0]
        if kind == "plain":
            prod = plain(t.init[1], cols)
            return lambda dst, r0, r1: prod(dst, r0 * cols, (r1 - r0) * cols)
        if kind == "concat":
            parts, first = [], 0
            for name, rows in t.init[1]:
                parts.append((first, first + rows, plain(name, cols)))
                first += rows

            def fill(dst, r0, r1):
                for a, b, prod in parts:
                    lo, hi = max(a, r0), min(b, r1)
                    if lo < hi:
                        prod(dst + (lo - r0) * cols * 2, (lo - a) * cols, (hi - lo) * cols)
            return fill
        if kind == "interleaved":
            name_a, name_b = t.init[1], t.init[2]
            scale, bias = init_scale(name_a, cols)
            sa, sb = tensor_seed(seed, name_a), tensor_seed(seed, name_b)
            rows_each = t.rows // 2
            return lambda dst, r0, r1: L.call("ps_init_interleaved_bf16", dst, rows_each, r0, r1 - r0, cols, sa,
                                              sb, scale, bias, stream)
        raise ValueError(f"unknown init {t.init!r}")

    def _generate_coded(self, staging_bytes: int) -> None:
        """Embedding table as bf16; every shard generated on the GPU and stored coded."""
        import torch

        from .hxcodec import HxShards
        stream = torch.cuda.current_stream().cuda_stream
        stage = torch.empty(staging_bytes, dtype=torch.uint8, device="cuda")
        emb = TensorSlot("embed", 0, self.spec.vocab_size, self.spec.d_model, ("plain", "embed"))
        fill = self.tensor_filler(emb, stream)
        step = max(1, staging_bytes // (emb.cols * 2))
        for r0 in range(0, emb.rows, step):
            r1 = min(emb.rows, r0 + step)
            fill(stage.data_ptr(), r0, r1)
            L.memcpy_async(self.embed + r0 * emb.cols * 2, stage.data_ptr(), (r1 - r0) * emb.cols * 2, stream)
            L.call("ps_stream_synchronize", stream)
        del stage
        kinds = {b.kind for b in self.layout.blobs.values()}
        self.hx = HxShards(self, kinds)

    def _generate(self, staging_bytes: int) -> None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
        stage = torch.empty(staging_bytes, dtype=torch.uint8, device="cuda")
        sptr = stage.data_ptr()

        def emit_rows(dst_host: int, t: TensorSlot) -> None:
            fill = self.tensor_filler(t, stream)
            step = max(1, staging_bytes // (t.cols * 2))
            for r0 in range(0, t.rows, step):
                r1 = min(t.rows, r0 + step)
                fill(sptr, r0, r1)
                L.memcpy_async(dst_host + r0 * t.cols * 2, sptr, (r1 - r0) * t.cols * 2, stream)
                L.call("ps_stream_synchronize", stream)

        for sid, blob in self.layout.blobs.items():
            for t in blob.tensors.values():
                emit_rows(self.base + blob.offset + t.offset, t)
        emb = TensorSlot("embed", 0, self.spec.vocab_size, self.spec.d_model, ("plain", "embed"))
        emit_rows(self.embed, emb)
        del stage
        torch.cuda.synchronize()
