"""ORACLE (test infrastructure only): fp32 CPU restatement of the decoder.

PARITY UNPINNED for logits/tokens: the reference (`shardplan`) computes no
numerics at all — "no weights are loaded and no GPU is required"
(pkg/README.md:20-22) — so there is no reference output to
pin this file to. It restates standard Llama-3 / Qwen3 decoder semantics on
the reference's shape conventions: attention weights Q, K, V, O
(`pkg/src/shardplan/model_graph.py:279-283`), a gated FFN with three matrices
(`:108-110`), a separate d x V output head (`:295-296`), RMSNorm, rotate-half
RoPE (Llama-3 frequency scaling for Llama-3.x), GQA, SwiGLU, greedy argmax.

Weights are regenerated from (seed, tensor name) by the C restatement of the
initialiser (oracle/c/weights.c), independent of the product's GPU init; the
tests check both bit-for-bit. Compute is fp32 on the bf16 weight values; the
KV cache is rounded to bf16 when stored, as the product stores it.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg use
this module.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import math
import os
import subprocess

import numpy as np
import torch

HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "_build", "liboracle.so")
        if not os.path.exists(path):
            subprocess.run(["make", "-C", HERE], check=True, capture_output=True)
        lib = C.CDLL(path)
        lib.oracle_init_uniform_bf16.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64,
                                                 C.c_float, C.c_float, C.c_int]
        lib.oracle_init_interleaved_bf16.argtypes = [C.c_void_p, C.c_longlong, C.c_int, C.c_uint64,
                                                     C.c_uint64, C.c_float, C.c_float]
        lib.oracle_bf16_to_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]
        _LIB = lib
    return _LIB


THREADS = max(1, min(32, os.cpu_count() or 1))


def seed_of(model_seed: int, name: str) -> int:
    return int.from_bytes(hashlib.sha256(f"{model_seed}:{name}".encode()).digest()[:8], "little")


def scale_bias(name: str, fan_in: int):
    leaf = name.rsplit(".", 1)[-1]
    if leaf.endswith("norm"):
        return 0.1, 1.0
    if leaf == "embed":
        return 1.0, 0.0
    return math.sqrt(3.0 / fan_in), 0.0


def bf16_bits(model_seed: int, name: str, rows: int, cols: int) -> np.ndarray:
    out = np.empty((rows, cols), np.uint16)
    sc, bi = scale_bias(name, cols)
    _lib().oracle_init_uniform_bf16(out.ctypes.data, out.size, seed_of(model_seed, name), 0,
                                    sc, bi, THREADS)
    return out


def interleaved_bits(model_seed: int, a: str, b: str, rows_each: int, cols: int) -> np.ndarray:
    out = np.empty((2 * rows_each, cols), np.uint16)
    sc, bi = scale_bias(a, cols)
    _lib().oracle_init_interleaved_bf16(out.ctypes.data, rows_each, cols, seed_of(model_seed, a),
                                        seed_of(model_seed, b), sc, bi)
    return out


def to_f32(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy((bits.astype(np.uint32) << 16).view(np.float32))


def weight(model_seed: int, name: str, rows: int, cols: int) -> torch.Tensor:
    return to_f32(bf16_bits(model_seed, name, rows, cols))


def bf16_round(x: torch.Tensor) -> torch.Tensor:
    return x.to(torch.bfloat16).to(torch.float32)


def inv_freq(theta: float, head_dim: int, scaling: dict | None) -> np.ndarray:
    base = 1.0 / (theta ** (np.arange(0, head_dim, 2, dtype=np.float64) / head_dim))
    if not scaling:
        return base
    f, lo, hi = scaling["factor"], scaling["low_freq_factor"], scaling["high_freq_factor"]
    orig = scaling["original_max_position_embeddings"]
    out = []
    for w in base:
        wavelen = 2 * math.pi / w
        if wavelen < orig / hi:
            out.append(w)
        elif wavelen > orig / lo:
            out.append(w / f)
        else:
            s = (orig / wavelen - lo) / (hi - lo)
            out.append((1 - s) * w / f + s * w)
    return np.array(out, np.float64)


def _bf16_tensor(bits: np.ndarray) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16)


class RefModel:
    """fp32 decoder with a per-request KV cache; hp = hyperparameter dict.

    lazy=True keeps weights as bf16 and upcasts each matrix to fp32 when it is
    used (large models: 2 bytes/param resident instead of 4)."""

    def __init__(self, hp: dict, seed: int = 0, threads: int | None = None, lazy: bool = False,
                 source=None):
        self.hp, self.seed, self.lazy = hp, seed, lazy
        if threads:
            torch.set_num_threads(threads)
        L, d, h, kv, hd = hp["n_layers"], hp["d_model"], hp["n_heads"], hp["n_kv_heads"], hp["head_dim"]
        ffn, V = hp["ffn_dim"], hp["vocab_size"]
        self.d, self.h, self.kvh, self.hd = d, h, kv, hd
        self.eps = hp.get("rms_eps", 1e-5)
        self.qk_norm = hp.get("qk_norm", False)
        get = source or (lambda name, rows, cols: _bf16_tensor(bf16_bits(seed, name, rows, cols)))

        def load(name, rows, cols):
            t = get(name, rows, cols)
            return t if lazy else t.float()

        self.embed = load("embed", V, d)
        self.layers = []
        self.moe = hp.get("moe")
        for i in range(L):
            lw = {
                "attn_norm": load(f"L{i}.attn_norm", 1, d)[0],
                "wq": load(f"L{i}.wq", h * hd, d),
                "wk": load(f"L{i}.wk", kv * hd, d),
                "wv": load(f"L{i}.wv", kv * hd, d),
                "wo": load(f"L{i}.wo", d, h * hd),
                "ffn_norm": load(f"L{i}.ffn_norm", 1, d)[0],
            }
            if self.moe:
                E, eff = self.moe["n_experts"], self.moe["expert_ffn_dim"]
                lw["router"] = load(f"L{i}.router", E, d)
                lw["experts"] = [(load(f"L{i}.e{e}.w_gate", eff, d), load(f"L{i}.e{e}.w_up", eff, d),
                                  load(f"L{i}.e{e}.w_down", d, eff)) for e in range(E)]
            else:
                lw["w_gate"] = load(f"L{i}.w_gate", ffn, d)
                lw["w_up"] = load(f"L{i}.w_up", ffn, d)
                lw["w_down"] = load(f"L{i}.w_down", d, ffn)
            if self.qk_norm:
                lw["q_norm"] = load(f"L{i}.q_norm", 1, hd)[0]
                lw["k_norm"] = load(f"L{i}.k_norm", 1, hd)[0]
            self.layers.append(lw)
        self.final_norm = load("final_norm", 1, d)[0]
        self.lm_head = load("lm_head", V, d)
        self.inv = torch.from_numpy(inv_freq(hp.get("rope_theta", 10000.0), hd,
                                             hp.get("rope_scaling")))

    @classmethod
    def from_host_weights(cls, hp: dict, hw, lazy: bool = True):
        """Same model over the bytes of an existing host weight blob (the CPU
        baseline reads what the GPU streams; tests check the bytes equal
        bf16_bits() of every tensor)."""
        views = {}
        for sid, blob in hw.layout.blobs.items():
            for name in blob.tensors:
                views[name] = (sid, name)
        h, kv, hd = hp["n_heads"], hp["n_kv_heads"], hp["head_dim"]

        def source(name, rows, cols):
            layer, _, leaf = name.partition(".")
            if name == "embed":
                return _bf16_tensor(hw.embed_view())
            if leaf in ("wq", "wk", "wv"):
                full = hw.host_view(*views[f"{layer}.wqkv"])
                lo = {"wq": 0, "wk": h * hd, "wv": (h + kv) * hd}[leaf]
                return _bf16_tensor(full[lo:lo + rows])
            if leaf in ("w_gate", "w_up"):
                full = hw.host_view(*views[f"{layer}.wgu"])
                return _bf16_tensor(full[0::2] if leaf == "w_gate" else full[1::2])
            if leaf == "w_down":
                return _bf16_tensor(hw.host_view(*views[f"{layer}.wdown"]))
            return _bf16_tensor(hw.host_view(*views[name]))
        return cls(hp, lazy=lazy, source=source)

    def _w(self, t: torch.Tensor) -> torch.Tensor:
        return t.float() if self.lazy else t

    def _moe(self, f, lw):
        """Qwen3-MoE block: softmax router, top-k, renormalised weights
        (norm_topk_prob), sum of the selected SwiGLU experts."""
        k = self.moe["top_k"]
        probs = torch.softmax(f @ self._w(lw["router"]).T, dim=-1)
        w, ids = torch.topk(probs, k, dim=-1)
        w = w / w.sum(-1, keepdim=True)
        out = torch.zeros_like(f)
        for t in range(f.shape[0]):
            for j in range(k):
                wg, wu, wd = (self._w(m) for m in lw["experts"][int(ids[t, j])])
                h = torch.nn.functional.silu(f[t] @ wg.T) * (f[t] @ wu.T)
                out[t] += w[t, j] * (h @ wd.T)
        return out

    def _rms(self, x, w):
        return x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + self.eps) * w

    def _rope(self, x, pos):
        # x [T, heads, hd]; rotate-half on pairs (i, i + hd/2); angles in fp64, table fp32
        ang = pos.to(torch.float64)[:, None] * self.inv[None, :]
        cos = torch.cos(ang).to(torch.float32)[:, None, :]
        sin = torch.sin(ang).to(torch.float32)[:, None, :]
        a, b = x[..., : self.hd // 2], x[..., self.hd // 2:]
        return torch.cat([a * cos - b * sin, b * cos + a * sin], dim=-1)

    def new_cache(self):
        return [{"k": torch.zeros(0, self.kvh, self.hd), "v": torch.zeros(0, self.kvh, self.hd)}
                for _ in self.layers]

    @torch.no_grad()
    def forward(self, tokens, cache) -> torch.Tensor:
        """Append `tokens` to one request's cache; returns fp32 logits [T, V]."""
        tokens = torch.as_tensor(np.asarray(tokens, np.int64))
        T = tokens.numel()
        p0 = cache[0]["k"].shape[0]
        pos = torch.arange(p0, p0 + T)
        x = self.embed[tokens].float()
        G = self.h // self.kvh
        for lw, c in zip(self.layers, cache):
            a = self._rms(x, self._w(lw["attn_norm"]))
            q = (a @ self._w(lw["wq"]).T).view(T, self.h, self.hd)
            k = (a @ self._w(lw["wk"]).T).view(T, self.kvh, self.hd)
            v = (a @ self._w(lw["wv"]).T).view(T, self.kvh, self.hd)
            if self.qk_norm:
                q = self._rms(q, self._w(lw["q_norm"]))
                k = self._rms(k, self._w(lw["k_norm"]))
            q, k = self._rope(q, pos), self._rope(k, pos)
            c["k"] = torch.cat([c["k"], bf16_round(k)])
            c["v"] = torch.cat([c["v"], bf16_round(v)])
            K = c["k"].repeat_interleave(G, dim=1)      # [S, h, hd]
            Vv = c["v"].repeat_interleave(G, dim=1)
            S = K.shape[0]
            scores = torch.einsum("thd,shd->hts", q, K) / math.sqrt(self.hd)
            mask = torch.arange(S)[None, :] > pos[:, None]
            scores = scores.masked_fill(mask[None], float("-inf"))
            o = torch.einsum("hts,shd->thd", torch.softmax(scores, -1), Vv).reshape(T, -1)
            x = x + o @ self._w(lw["wo"]).T
            f = self._rms(x, self._w(lw["ffn_norm"]))
            if self.moe:
                x = x + self._moe(f, lw)
            else:
                g, u = f @ self._w(lw["w_gate"]).T, f @ self._w(lw["w_up"]).T
                x = x + (torch.nn.functional.silu(g) * u) @ self._w(lw["w_down"]).T
        return self._rms(x, self._w(self.final_norm)) @ self._w(self.lm_head).T

    @torch.no_grad()
    def greedy(self, prompt, gen_len: int):
        cache = self.new_cache()
        logits = self.forward(prompt, cache)[-1:]
        toks, all_logits = [], [logits[0]]
        for _ in range(gen_len):
            t = int(torch.argmax(all_logits[-1]))
            toks.append(t)
            if len(toks) == gen_len:
                break
            all_logits.append(self.forward([t], cache)[0])
        return np.array(toks, np.int32), torch.stack(all_logits)

    @torch.no_grad()
    def teacher_forced(self, prompt, continuation):
        """Logits at each emitting position when the continuation is forced."""
        cache = self.new_cache()
        seq = list(np.asarray(prompt)) + list(np.asarray(continuation))[:-1]
        logits = self.forward(seq, cache)
        return logits[len(prompt) - 1:]


def hp_from_spec(spec, arch) -> dict:
    """Hyperparameters from a (ModelSpec, Arch) pair — plain values only."""
    return {"n_layers": spec.n_layers, "d_model": spec.d_model, "n_heads": spec.n_heads,
            "n_kv_heads": spec.n_kv_heads, "head_dim": spec.head_dim, "ffn_dim": spec.ffn_dim,
            "vocab_size": spec.vocab_size, "rope_theta": arch.rope_theta,
            "rope_scaling": arch.rope_scaling, "qk_norm": arch.qk_norm, "rms_eps": arch.rms_eps,
            "moe": None if spec.moe is None else {
                "n_experts": spec.moe.n_experts, "top_k": spec.moe.top_k,
                "expert_ffn_dim": spec.moe.expert_ffn_dim}}
