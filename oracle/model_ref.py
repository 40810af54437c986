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

Two uses: the plain fp32 model (`modes=None`) is the north_star's "fp32
reference" for the logit tolerance (max|d| / max|ref| <= 2e-2); with `modes`
(one of D / P / G per token, recorded by the engine per pass) it applies the
same bf16 rounding points as the GPU pass that computed each token, so greedy
ids can be required EXACTLY equal — what remains is fp32 summation order.

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
        lib.oracle_init_rowscaled_bf16.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64, C.c_uint64,
                                                   C.c_longlong, C.c_float]
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
    if name == "lm_head":   # heavy-tailed row norms (oracle/c/weights.c head_row_scale)
        _lib().oracle_init_rowscaled_bf16(out.ctypes.data, out.size, seed_of(model_seed, name), 0, cols, sc)
        return out
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
            expert, _, proj = leaf.rpartition(".")       # "e7.w_gate" -> ("e7", "w_gate")
            pre = f"{layer}.{expert}." if expert else f"{layer}."
            if proj in ("w_gate", "w_up"):
                full = hw.host_view(*views[pre + "wgu"])
                return _bf16_tensor(full[0::2] if proj == "w_gate" else full[1::2])
            if proj == "w_down":
                return _bf16_tensor(hw.host_view(*views[pre + "wdown"]))
            return _bf16_tensor(hw.host_view(*views[name]))
        return cls(hp, lazy=lazy, source=source)

    def _w(self, t: torch.Tensor) -> torch.Tensor:
        return t.float() if self.lazy else t

    def _moe(self, f, lw, g_rows):
        """Qwen3-MoE block: softmax router, top-k (ties -> lower id), renormalised weights
        (norm_topk_prob), sum of the selected SwiGLU experts in top-k slot order.
        Vectorised by expert: the rows routed to expert e go through it together.
        GEMM-pass rows feed the router and experts the bf16 rounding of `f` (the
        product's expert kernels read bf16 activations and keep h in fp32)."""
        k = self.moe["top_k"]
        fin = _round_rows(f, g_rows)
        probs = torch.softmax(fin @ self._w(lw["router"]).T, dim=-1)
        # stable descending sort: equal probabilities keep ascending expert ids
        order = torch.sort(probs, dim=-1, descending=True, stable=True)
        w, ids = order.values[:, :k], order.indices[:, :k]
        w = w / w.sum(-1, keepdim=True)
        contrib = torch.zeros(f.shape[0], k, f.shape[1])
        for e in torch.unique(ids).tolist():
            rows, slots = torch.nonzero(ids == e, as_tuple=True)
            wg, wu, wd = (self._w(m) for m in lw["experts"][e])
            xe = fin[rows]
            h = torch.nn.functional.silu(xe @ wg.T) * (xe @ wu.T)
            contrib[rows, slots] = w[rows, slots][:, None] * (h @ wd.T)
        out = contrib[:, 0]
        for j in range(1, k):
            out = out + contrib[:, j]
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

    def _attn_fp32(self, q, K, V, pos):
        """Exact fp32 causal softmax attention (the split-KV decode kernel's numerics)."""
        G = self.h // self.kvh
        K, V = K.repeat_interleave(G, dim=1), V.repeat_interleave(G, dim=1)
        S = K.shape[0]
        scores = torch.einsum("thd,shd->hts", q, K) / math.sqrt(self.hd)
        mask = torch.arange(S)[None, :] > pos[:, None]
        scores = scores.masked_fill(mask[None], float("-inf"))
        return torch.einsum("hts,shd->thd", torch.softmax(scores, -1), V).reshape(q.shape[0], -1)

    def _attn_tc(self, q, K, V, pos, block: int = 128):
        """The tcgen05 flash-attention kernel's numerics (csrc/attention_tc.cu): Q scaled
        by scale*log2(e) then rounded to bf16; per 128-key block a base-2 online softmax
        with the running max, P rounded to bf16 before P V, l summed from fp32 p, and
        the output multiplied by 1/l."""
        G = self.h // self.kvh
        T = q.shape[0]
        sl2 = np.float32(1.0 / math.sqrt(self.hd)) * np.float32(1.4426950408889634)
        qs = bf16_round(q * float(sl2)).permute(1, 0, 2)               # [h, T, hd]
        Kr = K.repeat_interleave(G, dim=1).permute(1, 0, 2)            # [h, S, hd]
        Vr = V.repeat_interleave(G, dim=1).permute(1, 0, 2)
        n_keys = int(pos.max()) + 1
        m = torch.full((self.h, T, 1), float("-inf"))
        l = torch.zeros(self.h, T, 1)
        o = torch.zeros(self.h, T, self.hd)
        for k0 in range(0, n_keys, block):
            k1 = min(n_keys, k0 + block)
            sc = qs @ Kr[:, k0:k1].transpose(1, 2)                      # [h, T, blk]
            mask = torch.arange(k0, k1)[None, :] > pos[:, None]
            sc = sc.masked_fill(mask[None], float("-inf"))
            m_new = torch.maximum(m, sc.amax(-1, keepdim=True))
            base = torch.where(torch.isinf(m_new), torch.zeros_like(m_new), m_new)
            corr = torch.exp2(m - base)
            p = torch.exp2(sc - base)
            l = l * corr + p.sum(-1, keepdim=True)
            o = o * corr + bf16_round(p) @ Vr[:, k0:k1]
            m = m_new
        inv = torch.where(l > 0, 1.0 / l, torch.zeros_like(l))
        return (o * inv).permute(1, 0, 2).reshape(T, -1)

    @torch.no_grad()
    def forward(self, tokens, cache, modes=None, logit_rows=None, perturb=None) -> torch.Tensor:
        """Append `tokens` to one request's cache; returns fp32 logits [rows, V].

        `modes` (one character per token, default all "D") mirrors where the GPU pass
        that computed each token rounds to bf16 (runtime/executor.py):
          "D"  decode-only GEMV pass: fp32 activations, fp32 split-KV attention;
          "P"  GEMV pass (<= 32 tokens) with the tcgen05 prefill attention: fp32
               activations, bf16 Q and P inside attention (`_attn_tc`);
          "G"  GEMM pass (> 32 tokens): the normalised input of every matmul rounded to
               bf16, tcgen05 attention with a bf16 output, SwiGLU output rounded to bf16.
        The residual stream, router logits, expert hidden states and the output head
        are fp32 in every mode; K and V are stored as bf16. `logit_rows`: rows whose
        logits to return (default all). `perturb` = (seed, eps): multiply the embedded
        inputs by (1 + eps * N(0, 1)) — the oracle's own numerical noise band: bf16
        rounding points amplify a 1e-7 input change to ~1e-3 of max|logit|,
        so positions whose top-2 margin lies inside that band have no well-defined
        bf16 argmax."""
        tokens = torch.as_tensor(np.asarray(tokens, np.int64))
        T = tokens.numel()
        modes = "D" * T if modes is None else modes
        if len(modes) != T or set(modes) - set("DPG"):
            raise ValueError(f"modes must be {T} characters of D/P/G")
        mode_arr = np.frombuffer(modes.encode(), np.uint8)
        g_rows = torch.from_numpy(mode_arr == ord("G"))
        tc_idx = torch.from_numpy(np.nonzero(mode_arr != ord("D"))[0])
        d_idx = torch.from_numpy(np.nonzero(mode_arr == ord("D"))[0])
        any_g = bool(g_rows.any())
        p0 = cache[0]["k"].shape[0]
        pos = torch.arange(p0, p0 + T)
        x = self.embed[tokens].float()
        if perturb is not None:
            g = torch.Generator().manual_seed(int(perturb[0]))
            x = x * (1 + float(perturb[1]) * torch.randn(x.shape, generator=g))
        for lw, c in zip(self.layers, cache):
            a = _round_rows(self._rms(x, self._w(lw["attn_norm"])), g_rows)
            q = (a @ self._w(lw["wq"]).T).view(T, self.h, self.hd)
            k = (a @ self._w(lw["wk"]).T).view(T, self.kvh, self.hd)
            v = (a @ self._w(lw["wv"]).T).view(T, self.kvh, self.hd)
            if self.qk_norm:
                q = self._rms(q, self._w(lw["q_norm"]))
                k = self._rms(k, self._w(lw["k_norm"]))
            q, k = self._rope(q, pos), self._rope(k, pos)
            c["k"] = torch.cat([c["k"], bf16_round(k)])
            c["v"] = torch.cat([c["v"], bf16_round(v)])
            o = torch.empty(T, self.h * self.hd)
            if len(d_idx):
                o[d_idx] = self._attn_fp32(q[d_idx], c["k"], c["v"], pos[d_idx])
            if len(tc_idx):
                o[tc_idx] = self._attn_tc(q[tc_idx], c["k"], c["v"], pos[tc_idx])
            o = _round_rows(o, g_rows)
            x = x + o @ self._w(lw["wo"]).T
            f = self._rms(x, self._w(lw["ffn_norm"]))
            if self.moe:
                x = x + self._moe(f, lw, g_rows)
            else:
                f = _round_rows(f, g_rows)
                g, u = f @ self._w(lw["w_gate"]).T, f @ self._w(lw["w_up"]).T
                hid = torch.nn.functional.silu(g) * u
                if any_g:
                    hid = _round_rows(hid, g_rows)
                x = x + hid @ self._w(lw["w_down"]).T
        if logit_rows is not None:
            x = x[torch.as_tensor(np.asarray(logit_rows, np.int64))]
        return self._rms(x, self._w(self.final_norm)) @ self._w(self.lm_head).T

    @torch.no_grad()
    def greedy(self, prompt, gen_len: int, modes=None):
        """Free-running greedy decode; `modes` (len(prompt) + gen_len - 1 characters,
        see `forward`) mirrors the passes that computed each position."""
        modes = modes or "D" * (len(prompt) + gen_len - 1)
        cache = self.new_cache()
        n = len(prompt)
        logits = self.forward(prompt, cache, modes[:n], logit_rows=[n - 1])
        toks, all_logits = [], [logits[0]]
        for i in range(gen_len):
            t = int(torch.argmax(all_logits[-1]))
            toks.append(t)
            if len(toks) == gen_len:
                break
            all_logits.append(self.forward([t], cache, modes[n + i])[0])
        return np.array(toks, np.int32), torch.stack(all_logits)

    @torch.no_grad()
    def teacher_forced(self, prompt, continuation, modes=None, perturb=None):
        """Logits at each emitting position when the continuation is forced, in one
        forward over prompt + continuation[:-1]; `modes` / `perturb` as in `forward`."""
        cache = self.new_cache()
        seq = list(np.asarray(prompt)) + list(np.asarray(continuation))[:-1]
        rows = list(range(len(prompt) - 1, len(seq)))
        return self.forward(seq, cache, modes, logit_rows=rows, perturb=perturb)


def greedy_parity(ref, prompt, got, modes, n_perturb: int = 1, eps: float = 1e-7) -> dict:
    """Token parity of a GPU greedy run `got` against the oracle, teacher-forced.

    The oracle runs with the GPU's per-pass rounding points (`modes`) and again with
    its inputs perturbed by `eps` (n_perturb seeds; 1e-7 ~ the fp32 summation-order noise of the GPU); the spread at each position is the
    oracle's own noise band (chaotic amplification by the bf16 rounding points). A
    position is DECIDED when the oracle's top-1 / top-2 margin exceeds twice that band
    and every perturbed run agrees on the argmax; there the GPU id must be the oracle's
    EXACTLY. At an undecided (near-tie) position the GPU id must be one of the tied
    candidates: its logit within twice the band of the top. Returns the counts and the
    mirrored logits (numpy [len(got), V])."""
    tf0 = ref.teacher_forced(prompt, got, modes).numpy()
    band = np.zeros(len(got))
    agree = np.ones(len(got), bool)
    top0 = tf0.argmax(1)
    for k in range(n_perturb):
        tfk = ref.teacher_forced(prompt, got, modes, perturb=(1000 + k, eps)).numpy()
        band = np.maximum(band, np.abs(tfk - tf0).max(1))
        agree &= tfk.argmax(1) == top0
    srt = np.sort(tf0, axis=1)
    margin = srt[:, -1] - srt[:, -2]
    decided = agree & (margin > 2 * band)
    got = np.asarray(got)
    exact_bad = [int(i) for i in np.nonzero(decided & (got != top0))[0]]
    tie_bad = [int(i) for i in np.nonzero(~decided)[0]
               if tf0[i, top0[i]] - tf0[i, got[i]] > 2 * band[i]]
    scale = float(np.abs(tf0).max())
    return {"positions": len(got), "decided": int(decided.sum()), "undecided": int((~decided).sum()),
            "exact_mismatch": exact_bad, "tie_mismatch": tie_bad,
            "equal": int((got == top0).sum()), "band_max": float(band.max()) / scale,
            "min_margin": float(margin.min()) / scale, "logits": tf0}


def _round_rows(x: torch.Tensor, rows: torch.Tensor) -> torch.Tensor:
    """bf16-round the rows of x selected by the boolean mask `rows`."""
    if not bool(rows.any()):
        return x
    if bool(rows.all()):
        return bf16_round(x)
    return torch.where(rows.view(-1, *([1] * (x.dim() - 1))), bf16_round(x), x)


def hp_from_spec(spec, arch) -> dict:
    """Hyperparameters from a (ModelSpec, Arch) pair — plain values only."""
    return {"n_layers": spec.n_layers, "d_model": spec.d_model, "n_heads": spec.n_heads,
            "n_kv_heads": spec.n_kv_heads, "head_dim": spec.head_dim, "ffn_dim": spec.ffn_dim,
            "vocab_size": spec.vocab_size, "rope_theta": arch.rope_theta,
            "rope_scaling": arch.rope_scaling, "qk_norm": arch.qk_norm, "rms_eps": arch.rms_eps,
            "moe": None if spec.moe is None else {
                "n_experts": spec.moe.n_experts, "top_k": spec.moe.top_k,
                "expert_ffn_dim": spec.moe.expert_ffn_dim}}
