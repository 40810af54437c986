"""The real pass: runs one tier's SchedulePlan on the GPU.

Replaces `simulate_schedule` (`pkg/src/shardplan/simulator.py:117-216`) inside
the generate loop. Per plan placement (`pkg/src/shardplan/planner.py:276-309`):

  VRAM_PINNED / GPU            weights (or the layer's KV cache) live in the
                               capped arena; kernels read them in place
  SYS_RAM / GPU / WEIGHTS_H2D  streamed through the copy-engine ring, one
                               row-aligned piece at a time, kernels per piece
  SYS_RAM / GPU / KV_H2D       the layer's KV home is pinned host memory: the
                               current prefix is streamed into the ring, new
                               rows are appended there and written back D2H
  SYS_RAM / CPU                no CPU backend exists: the GPU reads the shard
                               zero-copy from host-mapped memory (K8, no VRAM);
                               at T > 32 (GEMM passes) it is staged through the
                               ring instead, still inside the budget

Stream order is the plan's topological order with KV_i hoisted before
Attn_i (attention consumes the cache; SURVEY.md §7 hard part 4).

Numerics of a pass with T new tokens: the residual stream is fp32. T <= 32
uses the GEMV kernels on fp32 activations; larger T uses the tcgen05 GEMM
on bf16 activations. Attention: the split-KV decode kernel when every
request adds exactly one token (and T <= 32), else the causal varlen
flash-attention kernel.
"""

from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field

import numpy as np

from ..planning.faults import InfeasibleBudget, SpecError
from ..planning.graph import ShardKind, build_shards
from ..planning.placement import Residency, SchedulePlan, Streaming
from ..planning.vocab import Backend
from .migration import plan_relocation
from . import lib as L
from .arena import VramArena
from .model import Arch, HostWeights, rope_table
from .streamer import CopyRing, EventPool

GEMV_MAX_T = 32            # passes of <= 32 tokens keep fp32 activations (GEMV kernels)
GEMV_CORE_MAX_T = 8        # <= 8 tokens: CUDA-core bulk-copy GEMV; 9..32: tcgen05 one-pass GEMV
KV_PAGE_ROWS = 64          # positions per KV page (a 64-row TMA box never straddles pages)


class KvPagePool:
    """Paged KV cache bookkeeping: every layer's cache is a pool
    of `n_pages` pages of KV_PAGE_ROWS positions; the block table [slots, per_slot]
    names the physical page of each request's logical page and is shared by all layers
    (a request's pages have the same index in every layer's pool). Pages are taken on
    demand, lowest free index first (so one batch's live pages form the prefix [0, n)
    and move in one copy), or in a seeded random order (`seed`, tests: kernels and
    copies must honour the table). The pool holds B x ceil(context / 64) pages — the
    plan's KV shard (`pkg/src/shardplan/model_graph.py:299-304,331`) rounded up to
    whole pages."""

    def __init__(self, slots: int, per_slot: int, seed: int | None = None):
        self.slots, self.per_slot = slots, per_slot
        self.n_pages = slots * per_slot
        order = list(range(self.n_pages))
        if seed is not None:
            order = [int(i) for i in np.random.default_rng(seed).permutation(self.n_pages)]
        self.order = order
        self.reset()

    def reset(self) -> None:
        self.free = list(self.order)
        self.table = np.full((self.slots, self.per_slot), -1, np.int32)
        self.owned = [0] * self.slots
        self.version = getattr(self, "version", 0) + 1

    def ensure(self, slot: int, rows: int) -> bool:
        """Give `slot` pages for positions [0, rows); True when the table changed."""
        need = -(-rows // KV_PAGE_ROWS)
        if need > self.per_slot:
            raise SpecError(f"request slot {slot}: {rows} positions exceed the cache's "
                            f"{self.per_slot * KV_PAGE_ROWS}")
        changed = False
        while self.owned[slot] < need:
            self.table[slot, self.owned[slot]] = self.free.pop(0)
            self.owned[slot] += 1
            changed = True
        if changed:
            self.version += 1
        return changed

    def pages(self, slot: int, r0: int, r1: int) -> list:
        """Physical pages holding positions [r0, r1) of `slot`."""
        if r1 <= r0:
            return []
        return [int(p) for p in self.table[slot, r0 // KV_PAGE_ROWS:-(-r1 // KV_PAGE_ROWS)]]

    def live(self) -> list:
        return sorted(int(p) for s in range(self.slots) for p in self.table[s, :self.owned[s]])

    @staticmethod
    def runs(pages) -> list:
        """Sorted page ids -> [(first page, count)] of consecutive runs."""
        out = []
        for p in sorted(set(pages)):
            if out and out[-1][0] + out[-1][1] == p:
                out[-1][1] += 1
            else:
                out.append([p, 1])
        return [tuple(r) for r in out]


@dataclass
class PassSpec:
    """One pass: which request slots advance, by how many tokens, from where."""

    slots: list                 # request slot per participating request
    n_new: list                 # new tokens per participating request
    p0: list                    # position of the first new token per request
    ids: np.ndarray | None      # int32 [T] token ids (None: the previous pass's samples)
    sample: list                # participating-request indices that emit a token

    @property
    def T(self) -> int:
        return int(sum(self.n_new))

    @property
    def decode_only(self) -> bool:
        return all(n == 1 for n in self.n_new)


@dataclass
class PassStats:
    tier: int
    T: int
    bytes_streamed: int = 0      # every H2D byte of the pass (weights + KV windows)
    copies: int = 0
    kv_bytes: int = 0            # of which KV-cache pages (never coded)
    kv_writeback_bytes: int = 0
    zero_copy_bytes: int = 0
    kernel_calls: int = 0
    fetch_seqs: list = field(default_factory=list)   # (seq, bytes counted) until settled
    spec_hits: int = 0           # routed experts found prefetched (settled with the bytes)
    spec_routed: int = 0         # routed experts of the layers that had a prediction set
    spec_predicted: int = 0      # experts copied as predictions for a next layer
    spec_pred_bytes: int = 0     # their bytes


@dataclass
class Consumer:
    tensor: str | None          # tensor whose rows it consumes (None: runs between tensors)
    fn: object                  # fn(ptr, r0, r1)
    even_rows: bool = False     # piece boundaries on even rows (interleaved gate/up)
    reads: tuple = ()           # other (small) tensors it reads through `ptrs`


class Executor:
    def __init__(self, weights: HostWeights, arch: Arch, plans: dict, budget_bytes: float,
                 kv_slots: int, context_len: int, max_tokens: int,
                 chunk_bytes: int = 64 << 20, ring_cap: int = 1 << 30, kv_page_seed: int | None = None):
        spec = weights.spec
        self.moe = spec.moe
        self.spec, self.arch, self.w = spec, arch, weights
        self.plans = plans                       # tier -> SchedulePlan
        self.B = kv_slots
        self.cap = context_len
        self.Tmax = max_tokens
        self.shards = build_shards(spec, context_len, kv_slots)
        self.by_layer_kind = {(s.layer_index, s.kind): s for s in self.shards}
        n_loaded = C.c_int()
        L.call("ps_preload_kernels", C.byref(n_loaded))   # no lazy module load mid-pass
        self.shard_kind = {s.id: s.kind for s in self.shards}
        # routed-expert fetcher (copy-engine expert uploads in MoE decode); PS_MOE_FETCH=0 disables
        self.fetcher, self.fetch_seq = None, 0
        self.striper = None                           # runtime.striping.StripeLeader (set by Engine)
        self.fetch_enabled = os.environ.get("PS_MOE_FETCH", "1") != "0"
        # cache streamed / CPU-placed weight shards in budget the ring does not need
        # (PS_SPARE_PIN=0 runs the plan's residency exactly)
        self.spare_pin = os.environ.get("PS_SPARE_PIN", "1") != "0"
        self.spread_pins = os.environ.get("PS_SPREAD_PINS", "1") != "0"
        # ring kept for streaming, in pieces of chunk_cap: a GEMM (prefill) pass computes
        # for ms on each piece and wants a deep ring; a GEMV (decode) pass consumes a
        # piece in microseconds, so two keep the link busy and the rest of the budget
        # caches shards (config 2: 4 -> 2 pieces, one more attention shard cached,
        # 4.745 -> 4.80 tokens/s; config 4/5 prefill TTFT +1-16 % with 2, hence per tier)
        self.ring_keep_pieces = int(os.environ.get("PS_RING_KEEP_PIECES", "4"))
        self.ring_keep_pieces_decode = int(os.environ.get("PS_RING_KEEP_DECODE", "2"))
        self.spare_pinned = []
        self.expert_slots, self.expert_slot_bytes = 0, 0
        self._gapfill, self._piece_override, self._prefetched = None, {}, {}
        self._prefix_queue, self._prefix_dev = [], {}
        from collections import deque
        self._throttle_q = deque()
        L.lib()

        s = spec
        self.d, self.h, self.kv, self.hd = s.d_model, s.n_heads, s.n_kv_heads, s.head_dim
        self.qkv_rows = (self.h + 2 * self.kv) * self.hd
        self.ffn = s.ffn_dim if s.moe is None else 8   # MoE layers use the expert buffers below
        self.V = s.vocab_size
        self.row_elems = 2 * self.kv * self.hd
        self.row_bytes = self.row_elems * 2
        # paged KV cache: one page pool per layer, one block table for all layers
        self.pps = -(-self.cap // KV_PAGE_ROWS)              # pages per request slot
        self.kv_pages = KvPagePool(self.B, self.pps, kv_page_seed)
        self.page_bytes = KV_PAGE_ROWS * self.row_bytes
        self.kv_layer_bytes = self.kv_pages.n_pages * self.page_bytes
        self._bt_version = -1                                 # block-table version on the device

        self.cs = L.stream_create(high_priority=True)   # compute
        self.h2d = L.stream_create()                    # copy engine, host -> device
        self.d2h = L.stream_create()                    # KV write-back, token readback
        self.events = EventPool()
        # early head (one-token passes with a CPU-placed head, `_early_head`): a side
        # stream, the "x is final" flag (pass sequence) and the events around it
        self.hs = L.stream_create()
        self.head_seq = 0
        self._head_free = None    # dedicated events: the pool recycles its own within a pass
        self._ev_head_done, self._ev_head_free = L.event_create(False), L.event_create(False)

        # host KV homes: [layer][position][slot][K|V heads] bf16, pinned + mapped
        self.kv_host = L.host_alloc(max(1, s.n_layers * self.kv_layer_bytes), mapped=True)
        self.kv_len = [0] * self.B
        self.kv_vram: dict[int, int] = {}           # layer -> VRAM page pool
        self.kv_mode: dict[int, str] = {}
        self.kv_writeback: dict[int, int] = {}   # layer -> event of its last D2H append
        self.tok_events = [L.event_create(False) for _ in range(64)]

        self.arena = VramArena(budget_bytes)
        self._carve_persistent()
        # exponent-coded dense shards (runtime/wcomp.py) for GEMV passes that stream
        # them; every coded row carries its own base exponent and escapes (in-band)
        self.coded = getattr(weights, "coded", None)
        # host_format="coded": the coded shards are the only host copy, so every path reads them
        self.coded_only = getattr(weights, "host_format", "bf16") == "coded"
        self._coded_res_on = self.coded is not None and (self.coded_only or
                                                         os.environ.get("PS_CODED_RESIDENT", "1") != "0")
        self._coded_call = None
        # Huffman-coded exponents (runtime/hxcodec.py, ~10.4 bits/weight): dense shards
        # resident and streamed in hx form, expanded to bf16 piece by piece (PS_HX=0: off)
        self.hx = getattr(weights, "hx", None)
        self._hx_on = self.hx is not None and (self.coded_only or os.environ.get("PS_HX", "1") != "0")
        if self._hx_on:
            self.hx_lut = self.arena.alloc_high("hx_luts", self.hx.luts.nbytes)
            self._h2d_sync(self.hx_lut, self.hx.luts)
            self.hx_meta = self.arena.alloc_high("hx_blocks", 4096)
        self._zc_direct = False
        self.stage_zc = False
        self.stage_small = False
        self.persist_high = self.arena.high       # activations + ring are carved below, per tier
        self.residency: dict[int, tuple] = {}
        self.tier = None
        self.T_tier = 0
        self.chunk_cap, self.ring_cap = chunk_bytes, ring_cap
        # decode-tier piece size and the slack kept free beside the ring (<= 1/64 of the
        # budget): smaller decode pieces free budget for caching but shorten the ring's
        # look-ahead — config 2 measured 8.75 (64 MB / 32 MB slack) vs 8.74 (32 / 8) vs
        # 8.50 (16 / 8) tokens/s, config 4 360 vs 350: the defaults stay
        self.chunk_cap_decode = min(chunk_bytes, int(os.environ.get("PS_RING_CHUNK_DECODE", str(chunk_bytes))))
        self.ring_slack = int(os.environ.get("PS_RING_SLACK", str(32 << 20)))
        self.fixed_high = self.arena.high
        self.ring = None
        self.d2d_bytes = 0                          # tier switches: weights relocated in VRAM
        self.tracer = None                          # runtime.tracer.Tracer when attached
        self.stats: list[PassStats] = []
        self._unsettled: list[PassStats] = []   # passes with speculative fetches to settle
        self.host_tokens: list = []
        self._prev_sample_slots = None
        self._hx_res_on = self._hx_on
        self._choose_resident_form()

    def _choose_resident_form(self) -> None:
        """The form VRAM-resident dense shards take: bf16, 12-bit coded or hx. A coded form
        frees budget (0.75 / 0.64 x the bytes) that the decode tier may turn into more
        cached shards and fewer link bytes, but every use then pays a decode (12-bit: in
        the GEMV's inner loop; hx: an expansion pass). The cheapest form whose decode-tier
        link bytes are within 1 % of the best is taken: hx for Llama-3.1-8B @ 4 GB; bf16
        for the tiny model at 50 % (its one streamed shard, the head, fits in no form) and
        for Qwen3-30B-A3B (its dense shards fit as they are; a decode would sit on the
        per-layer routing chain). PS_HX_RESIDENT / PS_CODED_RESIDENT = 1 force a form, = 0
        exclude it; host_format='coded' has only the hx copy to upload."""
        hx_env = os.environ.get("PS_HX_RESIDENT", "auto")
        c12_env = os.environ.get("PS_CODED_RESIDENT", "auto")
        has_hx, has_c12 = self._hx_on, self._coded_res_on
        if self.coded_only or (has_hx and hx_env == "1"):
            self._hx_res_on, self._coded_res_on = has_hx, False
            self.resident_form = "hx" if has_hx else "bf16"
            return
        if has_c12 and c12_env == "1":
            self._hx_res_on, self._coded_res_on = False, True
            self.resident_form = "c12"
            return
        forms = ["bf16"]
        if has_c12 and c12_env != "0":
            forms.append("c12")
        if has_hx and hx_env != "0":
            forms.append("hx")
        dec = min((t for t in self.plans if t >= self.B), default=max(self.plans))
        T = min(dec, self.Tmax)
        k_frac = min(1.0, T * self.moe.top_k / self.moe.n_experts) if self.moe is not None else 1.0

        def link_bytes(form: str) -> float:
            self._hx_res_on, self._coded_res_on = form == "hx", form == "c12"
            pins = set(self.pins_for(dec))
            _, modes = self._plan_modes(self.plans[dec])
            total = 0.0
            for sid in modes:
                kind = self.shard_kind[sid]
                if sid in pins or kind is ShardKind.KV_CACHE:
                    continue
                nb = self.w.layout.blobs[sid].nbytes
                total += nb * k_frac if kind is ShardKind.MOE_EXPERT_GROUP else nb
            return total
        def fits(form: str) -> bool:   # the plan's own pins beside every tier's buffers
            self._hx_res_on, self._coded_res_on = form == "hx", form == "c12"
            up = lambda n: (n + 255) // 256 * 256  # noqa: E731
            for tier, plan in self.plans.items():
                high = (self.arena.capacity - self.persist_high) + \
                    sum(up(n) for _, _, n in self._activation_spec(min(tier, self.Tmax)))
                pinned, _ = self._plan_modes(plan)
                low = sum(up(self._phys_bytes(self.shards[p.shard_id])) for p in pinned)
                if low + high > self.arena.capacity:
                    return False
            return True
        feasible = [f for f in forms if fits(f)] or forms[-1:]
        lb = {f: link_bytes(f) for f in feasible}
        best = min(lb.values())
        pick = next(f for f in feasible if lb[f] <= 1.01 * best)
        self._hx_res_on, self._coded_res_on = pick == "hx", pick == "c12"
        self.resident_form = pick

    # ------------------------------------------------------------------ layout
    def _activation_spec(self, T: int) -> list:
        """(attribute, tag, bytes) of the activation buffers for passes of <= T tokens."""
        B, d = self.B, self.d
        t32 = min(T, GEMV_MAX_T)
        spec = [("x", "x", T * d * 4), ("qkv", "qkv", T * self.qkv_rows * 4),
                ("xn32", "xn32", t32 * d * 4), ("att32", "att32", t32 * self.h * self.hd * 4),
                ("hid32", "hid32", t32 * self.ffn * 4)]
        if T > GEMV_MAX_T:
            spec += [("xn16", "xn16", T * d * 2), ("att16", "att16", T * self.h * self.hd * 2),
                     ("hid16", "hid16", T * self.ffn * 2)]
        if T > GEMV_CORE_MAX_T:   # x planes + split-K partials of ps_gemv_tc
            spec.append(("tcws", "gemv_tc_ws", self._tc_workspace_bytes()))
        if self._hx_used() or (T > GEMV_MAX_T and (self._coded_prefill() or getattr(self, "_coded_res_on", False))):
            # one coded piece (streamed or VRAM-resident) expanded to bf16 for the GEMM, or,
            # with hx, for every pass (hx rows are only ever read through this buffer)
            spec.append(("expand", "coded_expand", self._expand_bytes()))
        spec += [("xs", "xs", B * d * 4), ("logits", "logits", B * self.V * 4)]
        # split-KV partials of ps_attn_decode (any pass with <= 32 tokens, whatever the tier)
        ws = L.attn_decode_workspace(B, self.h, self.hd, self.cap)
        spec.append(("ws", "attn_ws", max(1, ws) * 4))
        if self.moe is not None and self._hx_experts_on(T):
            # bf16 scratch experts the hx-coded routed experts expand into (blob layout)
            sid0 = next(iter(self.hx.experts))
            _, estride, _, _ = self._expert_geometry(sid0, self.shards[sid0].layer_index)
            spec.append(("hx_escratch", "hx_expert_scratch", self.moe.top_k * estride))
        if self.moe is not None:
            E, k, eff = self.moe.n_experts, self.moe.top_k, self.moe.expert_ffn_dim
            P = T * k
            n_ints = C.c_longlong()
            L.call("ps_moe_plan_ints", P, E, C.byref(n_ints))
            spec += [("m_logits", "moe_logits", T * E * 4), ("m_ids", "moe_ids", P * 4),
                     ("m_w", "moe_w", P * 4), ("m_plan", "moe_plan", n_ints.value * 4),
                     ("m_h", "moe_h", P * eff * 4), ("m_out", "moe_out", P * d * 4),
                     ("m_slotmap", "moe_slot_of_expert", E * 4),
                     # speculative prefetch: rank -> slot, predicted ids / weights, the two
                     # prediction sets, the next layer's normalised input
                     ("m_sor", "moe_slot_of_rank", P * 4), ("m_pids", "moe_pred_ids", 64 * 4),
                     ("m_pw", "moe_pred_w", 64 * 4), ("m_spec", "moe_spec_state", 2 * 64 * 4),
                     ("m_xp", "moe_pred_x", d * 4)]
        return spec

    def _hx_expand_bytes(self) -> int:
        """hx expansion buffer: <= 32 MB and 1/128 of the budget, >= one 64-row block of
        the widest matrix."""
        kmax = max((m.k for meta in self.hx.tensors.values() for _, m in meta.values() if m is not None),
                   default=256)
        return max(64 * kmax * 2, min(32 << 20, int(self.arena.capacity) // 128)) // 256 * 256

    def _hx_used(self) -> bool:
        return getattr(self, "_hx_on", False) and (getattr(self, "_hx_res_on", False) or self._hx_stream_on())

    def _expand_bytes(self) -> int:
        """The bf16 expansion buffer: the hx size when hx rows are in use, else (12-bit
        coded GEMM pieces) one ring piece at most and at most 1/64 of the budget (small
        budgets keep their ring)."""
        if self._hx_used():
            return self._hx_expand_bytes()
        return max(64 << 10, min(self.chunk_cap, int(self.arena.capacity) // 64)) // 256 * 256

    def _hx_prefill_experts(self, sid: int) -> bool:
        """GEMM passes stream this MoE group's experts hx-coded and expand them in VRAM
        (PS_HX_PREFILL_EXPERTS=0: bf16). Needs the expansion buffer to hold one expert."""
        if not (getattr(self, "_hx_on", False) and self.expand and os.environ.get("PS_HX_PREFILL_EXPERTS", "1") != "0"):
            return False
        hxg = getattr(self.hx, "experts", {}).get(sid)
        if hxg is None:
            return False
        layer = self.shards[sid].layer_index
        return self._expand_bytes() >= self._expert_geometry(sid, layer)[1] and self.ring.capacity >= hxg["stride"]

    def _coded_prefill(self) -> bool:
        """GEMM (prefill) passes stream coded pieces and expand them in VRAM (PS_CODED_PREFILL)."""
        return getattr(self, "coded", None) is not None and (
            getattr(self, "coded_only", False) or os.environ.get("PS_CODED_PREFILL", "1") != "0")

    def _tc_workspace_bytes(self) -> int:
        """ps_gemv_tc workspace: the x planes of the widest K, plus split-K partials up to
        the size that leaves every shape its best split (~4.9 MB), capped at 1/128 of the
        budget (small budgets run fewer splits; results differ only in summation order)."""
        if getattr(self, "_tcws_bytes", None) is None:
            s = self.spec
            kmax = max(self.d, self.h * self.hd, s.ffn_dim if s.moe is None else self.d)
            planes = (3 * 32 * kmax * 2 + 255) // 256 * 256
            ideal = C.c_longlong()
            best = planes
            for K in {self.d, self.h * self.hd, s.ffn_dim if s.moe is None else self.d}:
                for N in list(range(128, 40064, 128)) + [self.qkv_rows, 2 * s.ffn_dim, self.V]:
                    L.call("ps_gemv_tc_workspace", N, K, C.byref(ideal))
                    best = max(best, ideal.value)
            self._tcws_bytes = int(max(planes, min(best, int(self.arena.capacity) // 128))) // 256 * 256
        return self._tcws_bytes

    def _carve_activations(self, T: int) -> None:
        """Activation buffers for passes of <= T tokens (re-carved per tier, so a
        decode tier holds only what the plan's activation scratch allows)."""
        self.xn16 = self.att16 = self.hid16 = self.tcws = self.expand = self.hx_escratch = 0
        for attr, tag, n in self._activation_spec(T):
            setattr(self, attr, self.arena.alloc_high(tag, n))
        self.ws_floats = L.attn_decode_workspace(self.B, self.h, self.hd, self.cap)

    def _carve_persistent(self) -> None:
        """Small buffers whose content outlives a pass (tokens, rope table)."""
        a, T, B = self.arena, self.Tmax, self.B
        self.i_ids = a.alloc_high("ids", T * 4)
        self.i_pos = a.alloc_high("pos", T * 4)
        self.i_req = a.alloc_high("req", T * 4)
        self.i_meta = a.alloc_high("meta", 4 * (4 * B + 4))
        self.i_rows = a.alloc_high("sample_rows", B * 4)
        self.i_bt = a.alloc_high("kv_block_table", B * self.pps * 4)
        self.i_tok_ring = a.alloc_high("sample_tok", 8 * B * 4)   # 8 rotating slots
        self.head_flag = a.alloc_high("head_flag", 256)
        L.call("ps_memset_async", self.head_flag, 0, 256, self.cs)
        self.tok_slot = 0
        self.i_tok = self.i_tok_ring
        rope = rope_table(self.arch, self.hd, self.cap)
        self.rope = a.alloc_high("rope", rope.nbytes)
        self.host_stage_bytes = max(1 << 20, rope.nbytes, T * 4 + 4096)
        self.host_stage = L.host_alloc(self.host_stage_bytes, mapped=False)
        self._h2d_sync(self.rope, rope)
        self.host_tok = L.host_alloc(4 * B * 4096, mapped=False)
        self.host_tok_i = 0

    def _h2d_sync(self, dst: int, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr)
        src = arr.ctypes.data
        for o in range(0, arr.nbytes, self.host_stage_bytes):
            n = min(self.host_stage_bytes, arr.nbytes - o)
            L.call("ps_stream_synchronize", self.cs)
            C.memmove(self.host_stage, src + o, n)
            L.memcpy_async(dst + o, self.host_stage, n, self.cs)
        L.call("ps_stream_synchronize", self.cs)

    def _phys_bytes(self, shard) -> int:
        if shard.kind is ShardKind.KV_CACHE:
            return self.kv_layer_bytes
        if self.hx_resident(shard.id):
            return self.hx.shard_bytes[shard.id]
        if self.coded_resident(shard.id):
            return self.coded.shard_bytes[shard.id]
        return self.w.layout.blobs[shard.id].nbytes

    def _hx_stream_on(self) -> bool:
        """Stream hx pieces: when the expand buffer takes runs of useful size (>= 4 MB; a
        30 MB budget's 1/128 would expand a piece in ~100 tiny launches — such budgets
        stream the 12-bit rows, read directly by the GEMV), or on an hx-only host copy
        (PS_HX_STREAM=1 / 0 forces it)."""
        if not self._hx_on:
            return False
        env = os.environ.get("PS_HX_STREAM")
        if env in ("0", "1") and not self.coded_only:
            return env == "1"
        return self.coded_only or self._hx_expand_bytes() >= (4 << 20) or self.coded is None

    def _hx_experts_on(self, T: int) -> bool:
        """One-token MoE passes fetch routed experts hx-coded (PS_HX_EXPERTS=0: off)."""
        return (T == 1 and self._hx_on and bool(getattr(self.hx, "experts", None)) and self.fetch_enabled and
                os.environ.get("PS_HX_EXPERTS", "1") != "0")

    def _spec_n(self, T: int) -> int:
        """_spec_want(T) when the carved expert slots have room for the two prediction
        sets, else 0."""
        S = self._spec_want(T)
        if S and getattr(self, "expert_slot_count", 0) < T * self.moe.top_k + 2 * S:
            return 0
        return S

    def _spec_want(self, T: int) -> int:
        """Experts predicted per fetched MoE layer for the next one (speculative pre-gated
        prefetch, csrc/fetcher.cu; PS_MOE_SPEC, default 2, 0: off): one-token passes that
        fetch hx-coded experts. The next layer's router applied to this layer's
        post-attention state names one of the next layer's routed experts with ~90 % of
        its top-2 picks on config 3 (bench `moe_prefetch`; sweep in DESIGN.md §5b)."""
        if self.moe is None or not self._hx_experts_on(T):
            return 0
        return max(0, min(int(os.environ.get("PS_MOE_SPEC", "2")), self.moe.top_k, 64))

    def _early_head_plan(self, T: int, R: int):
        """(final_norm ptr, head W ptr, ldw, coded) when this pass should read its CPU-placed
        head early, else None. One-token passes of one sampled row whose head is read
        zero-copy: the head GEMV is launched on a side stream at the start of the pass
        (ps_gemv_head_early, half the SMs), streaming the head rows from host memory while
        the layers compute on the other SMs, and computes once the compute stream flags x
        final — meant to overlap the zero-copy read (~0.5 ms for config 1's 25 MB head)
        with the ~0.25 ms of layers. Measured slower (1415 -> 1306 tokens/s on config 1):
        the bulk-copy GEMV's stages are sized for 4096-column rows, so on the tiny head
        (512 columns) half the SMs hold ~1 MB in flight and then stream the rest at half
        rate. Off by default (PS_HEAD_EARLY=1 turns it on; tests keep it exact)."""
        if T > GEMV_CORE_MAX_T or R != 1 or os.environ.get("PS_HEAD_EARLY", "0") != "1" or \
                self.striper is not None or (self.stage_zc and self.stage_small):
            return None
        sid = self.by_layer_kind[(self.spec.n_layers, ShardKind.OUTPUT_HEAD)].id
        if self.residency.get(sid, ("", 0))[0] != "zerocopy":
            return None
        blob = self.w.layout.blobs[sid]
        if (self.coded is not None and sid in self.coded.tensors and getattr(self.coded, "mapped", False) and
                (self.coded_only or os.environ.get("PS_CODED_ZEROCOPY", "1") != "0")):
            meta = self.coded.tensors[sid]
            base = self.coded.shard_ptr(sid)
            off, rb, coded = meta["lm_head"]
            return (base + meta["final_norm"][0], base + off, rb if coded else self.d, 1 if coded else 0,
                    self.coded.shard_bytes[sid])
        if not self.w.base:
            return None
        base = self.w.shard_ptr(sid)
        return (base + blob.tensors["final_norm"].offset, base + blob.tensors["lm_head"].offset, self.d, 0,
                blob.nbytes)

    def _zc_readable(self, sid: int) -> bool:
        """A CPU-placed shard can be read zero-copy: the bf16 blob or its 12-bit coded
        copy is on the host (an hx-only host copy must be staged through the ring)."""
        if self.w.base:
            return True
        return (self.coded is not None and sid in self.coded.tensors and getattr(self.coded, "mapped", False))

    def hx_resident(self, sid: int) -> bool:
        """Dense shards held in VRAM hx-coded (~0.65 x bf16), expanded per use
        (`_choose_resident_form`)."""
        return self._hx_on and getattr(self, "_hx_res_on", True) and sid in self.hx.tensors

    def phys_bytes(self, sid: int) -> int:
        """VRAM bytes shard `sid` takes when resident (the migration model's size)."""
        return self._phys_bytes(self.shards[sid])

    def coded_resident(self, sid: int) -> bool:
        """Dense weight shards live in VRAM in their exponent-coded form (runtime/wcomp.py,
        0.75 x the bytes): GEMV passes read the coded rows, GEMM passes expand them to bf16
        piece by piece. The freed budget caches more shards (spare pins), so fewer bytes
        cross the link per token. MoE expert groups stay bf16 (PS_CODED_RESIDENT=0: all)."""
        return (self._coded_res_on and sid in self.coded.tensors and not self.hx_resident(sid) and
                self.shard_kind[sid] is not ShardKind.MOE_EXPERT_GROUP)

    def _pinned_bytes(self, plan: SchedulePlan) -> int:
        return sum((self._phys_bytes(self.shards[p.shard_id]) + 255) // 256 * 256
                   for p in plan.placements if p.residency is Residency.VRAM_PINNED)

    def _kv_host_ptr(self, layer: int) -> int:
        return self.kv_host + layer * self.kv_layer_bytes

    def _copy_pages(self, dst_pool: int, src_pool: int, runs: list, stream: int) -> int:
        """Copy page runs between two pools with the same page offsets; returns bytes."""
        n = 0
        for p, c in runs:
            L.memcpy_async(dst_pool + p * self.page_bytes, src_pool + p * self.page_bytes,
                           c * self.page_bytes, stream)
            n += c * self.page_bytes
        return n

    def kv_live_pages(self) -> int:
        """Pages each layer's cache holds for the live requests (what a tier switch moves)."""
        return len(self.kv_pages.live())

    def reset_requests(self) -> None:
        """A new request batch: every page back to the free list, every slot empty."""
        self.kv_pages.reset()
        self.kv_len = [0] * self.B

    def _sync_block_table(self) -> None:
        """Upload the block table when it changed (stream-ordered, kernel parameter
        copies of <= 4000 bytes: no host sync, nothing queued behind weight copies)."""
        if self._bt_version == self.kv_pages.version:
            return
        flat = self.kv_pages.table.reshape(-1)
        step = 1000
        for i in range(0, len(flat), step):
            self._upload(self.i_bt + 4 * i, flat[i:i + step])
        self._bt_version = self.kv_pages.version

    # --------------------------------------------------------------- residency
    def _plan_modes(self, plan) -> tuple:
        """(pinned placements in pin order, {shard id: 'stream' | 'zerocopy'} of the rest)."""
        pinned = sorted((p for p in plan.placements if p.residency is Residency.VRAM_PINNED),
                        key=lambda p: (self.shards[p.shard_id].priority,
                                       self.shards[p.shard_id].layer_index, p.shard_id))
        modes = {}
        for p in plan.placements:
            if p.residency is Residency.VRAM_PINNED:
                continue
            if p.exec_backend is Backend.CPU:
                modes[p.shard_id] = "zerocopy"
            elif p.streaming in (Streaming.WEIGHTS_H2D, Streaming.KV_H2D, Streaming.WEIGHTS_AND_KV):
                modes[p.shard_id] = "stream"
            else:
                raise SpecError(f"unsupported placement {p}")
        return pinned, modes

    def _slot_bytes(self, T: int, modes: dict, free: int) -> tuple:
        """(slot count, slot bytes) of the routed-expert fetcher at this tier (0, 0: none)."""
        if self.moe is None or T > GEMV_MAX_T or not self.fetch_enabled:
            return 0, 0
        groups = [sid for sid, m in modes.items()
                  if m == "stream" and self.shard_kind[sid] is ShardKind.MOE_EXPERT_GROUP]
        if not groups:
            return 0, 0
        _, _, _, ebytes = self._expert_geometry(groups[0], self.shards[groups[0]].layer_index)
        slot = (ebytes + 255) // 256 * 256
        n = min(self.moe.n_experts, T * self.moe.top_k)
        if (n + 2 * self._spec_want(T)) * slot <= free // 4:
            n += 2 * self._spec_want(T)   # the two prediction sets, when they fit as well
        if n * slot > free // 4:
            return 0, 0
        return n, slot

    def pins_for(self, tier: int) -> list:
        """Shard ids carved into VRAM at `tier`, in carve order: the plan's pinned
        set in pin order, then the *spare pins* — streamed or CPU-placed weight
        shards cached in budget the plan reserved as double-buffer scratch
        (2 x the largest streamed shard, `pkg/src/shardplan/planner.py:132-159`)
        but the piece-wise ring (4 pieces ahead) does not need; first-fit
        decreasing by link bytes saved per token. Pure: a function of the plan,
        the layout and the budget, so the migration model can predict switches."""
        plan = self.plans[tier]
        T = min(tier, self.Tmax)
        pinned, modes = self._plan_modes(plan)
        out = [p.shard_id for p in pinned]
        if not self.spare_pin:
            return out
        up = lambda n: (n + 255) // 256 * 256  # noqa: E731
        high = (self.arena.capacity - self.persist_high) + sum(up(n) for _, _, n in self._activation_spec(T))
        low = sum(up(self._phys_bytes(self.shards[sid])) for sid in out)
        free = self.arena.capacity - high - low
        n_slots, slot = self._slot_bytes(T, modes, free)
        # a GEMM pass stages zero-copy KV through the ring too
        kv_staged = ("stream", "zerocopy") if T > GEMV_MAX_T else ("stream",)
        kv_streams = any(m in kv_staged and self.shards[sid].kind is ShardKind.KV_CACHE
                         for sid, m in modes.items())
        keep = self.ring_keep_pieces if T > GEMV_MAX_T else self.ring_keep_pieces_decode
        cc = self.chunk_cap if T > GEMV_MAX_T else self.chunk_cap_decode
        ring_keep = min(self.ring_cap, keep * cc + (self.kv_layer_bytes if kv_streams else 0))
        spare = free - n_slots * slot - ring_keep - min(self.ring_slack, self.arena.capacity // 64)
        if spare <= 0:
            return out
        k_frac = 1.0
        if self.moe is not None:
            k_frac = min(1.0, T * self.moe.top_k / self.moe.n_experts)

        def value(sid):   # link bytes saved per token per VRAM byte
            return k_frac if self.shard_kind[sid] is ShardKind.MOE_EXPERT_GROUP else 1.0
        # equal value per byte packs best largest-first (first-fit decreasing); among equal
        # shards, layers in bit-reversed order (0, L/2, L/4, 3L/4, ...): the cached layers
        # spread over the pass, so no long run of resident compute (at batch 32, ~1 ms a
        # layer) outlasts the ring's look-ahead and idles the link
        nbits = max(1, (self.spec.n_layers - 1).bit_length())

        def spread(layer):
            return int(format(layer, f"0{nbits}b")[::-1], 2) if self.spread_pins else layer
        cands = sorted((sid for sid in modes if self.shard_kind[sid] is not ShardKind.KV_CACHE),
                       key=lambda sid: (-value(sid), -self._phys_bytes(self.shards[sid]),
                                        self.shards[sid].priority, spread(self.shards[sid].layer_index), sid))
        for sid in cands:
            b = up(self._phys_bytes(self.shards[sid]))
            if b <= spare:
                out.append(sid)
                spare -= b
        return out

    def set_tier(self, tier: int) -> int:
        """Make `tier`'s plan resident (the paper's SetupForSched); returns the
        bytes moved. The reference charges this 0; the engine
        charges it to the pass that follows."""
        if tier == self.tier:
            return 0
        plan = self.plans[tier]
        moved = 0
        live = self.kv_pages.runs(self.kv_pages.live())
        # 1. every VRAM KV cache goes home first (content is authoritative): its live pages
        for layer, dev in self.kv_vram.items():
            moved += self._copy_pages(self._kv_host_ptr(layer), dev, live, self.cs)
        L.call("ps_stream_synchronize", self.cs)
        self.synchronize()   # the ring and every stream must be idle before re-carving
        # 2. re-carve the pinned region in pin order; weights whose slot is unchanged
        #    stay, weights resident at another offset are relocated device to device
        old = {sid: (r[1], self._phys_bytes(self.shards[sid]))
               for sid, r in self.residency.items() if r[0] == "pinned"}
        self.ring = None
        self.arena.high = self.persist_high        # drop the previous tier's activations + ring
        self.arena.reset_low()                     # ... and its pinned region
        self.T_tier = min(tier, self.Tmax)
        pins = self.pins_for(tier)                 # plan pins, then spare pins
        _, modes = self._plan_modes(plan)
        self._carve_activations(self.T_tier)
        self.fixed_high = self.arena.high
        self.residency, self.kv_vram, self.kv_mode = {}, {}, {}
        plan_pinned = {p.shard_id for p in plan.placements if p.residency is Residency.VRAM_PINNED}
        self.spare_pinned = [sid for sid in pins if sid not in plan_pinned]
        new = {}
        for sid in pins:
            s = self.shards[sid]
            dev = self.arena.alloc_low(f"pin{s.id}", self._phys_bytes(s))
            if s.kind is ShardKind.KV_CACHE:
                self.kv_vram[s.layer_index] = dev
                self.kv_mode[s.layer_index] = "pinned"
            else:
                new[sid] = (dev, self._phys_bytes(s))
                self.residency[s.id] = ("pinned", dev)
        d2d, h2d = plan_relocation(old, new)
        for _, src, dst, nbytes in d2d:          # before anything lands on a source
            L.memcpy_async(dst, src, nbytes, self.cs)
            self.d2d_bytes += nbytes
        for sid in h2d:
            dev, nbytes = new[sid]
            src = (self.hx.shard_ptr(sid) if self.hx_resident(sid) else
                   self.coded.shard_ptr(sid) if self.coded_resident(sid) else self.w.shard_ptr(sid))
            L.memcpy_async(dev, src, nbytes, self.cs)
            moved += nbytes
        for layer, dev in self.kv_vram.items():
            moved += self._copy_pages(dev, self._kv_host_ptr(layer), live, self.cs)
        for sid, mode in modes.items():
            if sid in self.residency:
                continue
            s = self.shards[sid]
            if s.kind is ShardKind.KV_CACHE:
                self.kv_mode[s.layer_index] = mode
            else:
                if mode == "zerocopy" and not self._zc_readable(sid):
                    mode = "stream"      # no host form the SMs can read (hx-only host copy)
                self.residency[sid] = (mode, 0)
        self._carve_ring(tier, modes)
        L.call("ps_stream_synchronize", self.cs)
        self.tier = tier
        return moved

    def _carve_ring(self, tier: int, modes: dict | None = None) -> None:
        """The staging ring takes what the tier's pinned set leaves (<= ring_cap).

        A tier that streams nothing (every shard pinned or zero-copy) needs no
        ring; one that streams needs room for a layer's KV prefix plus a few
        pieces, else the budget is infeasible for this executor."""
        self.arena.high = self.fixed_high
        self.arena.high_marks.pop("ring", None)
        self.arena.high_marks.pop("expert_slots", None)
        self._carve_expert_slots(tier, modes)
        free = self.arena.free_bytes
        ring_bytes = max(0, min(self.ring_cap, free)) // 256 * 256
        gemm = self.T_tier > GEMV_MAX_T   # GEMM passes cannot read host memory: staging is required
        staged = ("stream", "zerocopy") if gemm else ("stream",)
        kv_win = self.kv_layer_bytes if any(m in staged for m in self.kv_mode.values()) else 0
        # pieces of <= 1/6 of what the KV window leaves, so three always fit beside it
        cc = self.chunk_cap if gemm else self.chunk_cap_decode
        self.chunk = min(cc, max(1 << 16, (ring_bytes - kv_win) // 6 // 256 * 256))
        need = kv_win + 3 * self.chunk
        streams = kv_win > 0 or any(m in staged for m, _ in self.residency.values())
        # CPU-placed shards go through the ring when it fits in passes of 9..32 tokens:
        # read once, not per 8 tokens. One-token passes keep reading them zero-copy:
        # staging would buy the copy engine (55.6 vs ~50 GB/s) and overlap with the
        # resident layers, but config 1's 8 MB ring cuts its 25 MB head into ~19 pieces
        # (a GEMV launch and an event wait each) and ends programmatic dependent launch:
        # 1337 -> 1121 tokens/s measured (PS_STAGE_ZC=1 turns it on). A budget whose ring
        # cannot hold that keeps reading them zero-copy.
        small = self.stage_small = os.environ.get("PS_STAGE_ZC", "0") == "1"
        self.stage_zc = (self.T_tier > GEMV_CORE_MAX_T or small) and ring_bytes >= need and \
            any(m == "zerocopy" and self.shard_kind[sid] is not ShardKind.MOE_EXPERT_GROUP
                for sid, (m, _) in self.residency.items())
        if streams and ring_bytes < need:
            raise InfeasibleBudget(float(self.arena.capacity),
                                   float(self.arena.capacity - free + need), "copy-engine ring")
        if ring_bytes == 0:
            self.ring = None
            return
        self.ring = CopyRing(self.arena.alloc_high("ring", ring_bytes), ring_bytes, self.h2d,
                             self.events)
        self.ring.tracer = self.tracer
        self.ring.striper = self.striper

    # ------------------------------------------------- routed-expert fetcher
    def _expert_geometry(self, sid: int, layer: int) -> tuple:
        """(offset of expert 0, stride between experts, offset of wdown in an
        expert, bytes of one expert) inside a MoE group's blob."""
        blob = self.w.layout.blobs[sid]
        e0 = blob.tensors[f"L{layer}.e0.wgu"]
        E = self.moe.n_experts
        stride = blob.tensors[f"L{layer}.e1.wgu"].offset - e0.offset if E > 1 else blob.nbytes - e0.offset
        wd = blob.tensors[f"L{layer}.e0.wdown"]
        nbytes = wd.offset + wd.rows * wd.cols * 2 - e0.offset
        return e0.offset, stride, wd.offset - e0.offset, nbytes

    def _carve_expert_slots(self, tier: int, modes: dict | None = None) -> None:
        """VRAM slots for the routed experts of one MoE layer in a decode pass
        (min(E, T*k) experts), carved before the ring so fetcher copies never
        race the ring's reuse. Used when a decode tier streams expert groups and
        the slots take at most a quarter of the free budget (decided before spare
        pinning, `_slot_bytes`); otherwise the expert kernels read the routed
        experts zero-copy."""
        self.expert_slots, self.expert_slot_bytes, self.expert_slot_count = 0, 0, 0
        if modes is None:
            modes = {sid: m for sid, (m, _) in self.residency.items() if m != "pinned"}
        plan_free = self.arena.free_bytes + sum((self._phys_bytes(self.shards[sid]) + 255) // 256 * 256
                                                for sid in getattr(self, "spare_pinned", []))
        n, slot = self._slot_bytes(self.T_tier, modes, plan_free)
        if not n:
            return
        # the spare pins were sized around these slots
        self.expert_slots = self.arena.alloc_high("expert_slots", n * slot)
        self.expert_slot_bytes, self.expert_slot_count = slot, n
        if self.fetcher is None:
            out = C.c_void_p()
            L.call("ps_fetcher_create", self.moe.n_experts, C.byref(out))
            self.fetcher = out.value

    def _fetch_debug(self, layer, seq, P, E, host, stride, ebytes, slots, sb) -> None:
        """PS_FETCH_DEBUG=1: synchronise and check ids, slot map and slot bytes."""
        import torch
        L.call("ps_stream_synchronize", self.cs)
        ids = np.zeros(P, np.int32)
        L.call("ps_memcpy_async", ids.ctypes.data, self.m_ids, P * 4, self.cs)
        smap = np.zeros(E, np.int32)
        L.call("ps_memcpy_async", smap.ctypes.data, self.m_slotmap, E * 4, self.cs)
        L.call("ps_stream_synchronize", self.cs)
        routed = sorted(set(int(i) for i in ids))
        bad = [i for i in ids if not 0 <= i < E]
        ok_map = all(smap[e] == (routed.index(e) if e in routed else -1) for e in range(E)) if not bad else False
        mism = []
        if not bad:
            for r, e in enumerate(routed):
                got = np.zeros(ebytes, np.uint8)
                L.call("ps_memcpy_async", got.ctypes.data, slots + r * sb, ebytes, self.cs)
                L.call("ps_stream_synchronize", self.cs)
                want = np.ctypeslib.as_array((C.c_uint8 * ebytes).from_address(host + e * stride))
                if not np.array_equal(got, want):
                    mism.append(e)
        print(f"[fetch-debug] layer {layer} seq {seq} ids {ids.tolist()} bad {bad} map_ok {ok_map} "
              f"slot_mismatch {mism} stats {self.fetcher_stats()}", flush=True)

    def _throttle_host(self, window: int = 4) -> None:
        """Keep the host at most `window` fetched MoE layers ahead of the GPU. A host
        that runs further fills the driver's command queue and then blocks *inside* a
        launch call, holding the context lock the fetcher thread needs for its
        cudaMemcpyAsync — which delays the copies the GPU is spinning on. Polling an
        event (cudaEventQuery, no lock held while sleeping) keeps the queue shallow."""
        import time
        q = self._throttle_q
        ev = self.events.next()
        L.call("ps_event_record", ev, self.cs)
        q.append(ev)
        while len(q) > window:
            head = q[0]
            while not L.event_query(head):
                time.sleep(20e-6)
            q.popleft()

    def fetcher_stats(self) -> dict:
        if self.fetcher is None:
            return {}
        n, b, err = C.c_longlong(), C.c_longlong(), C.c_int()
        L.call("ps_fetcher_info", self.fetcher, None, None, C.byref(n), C.byref(b), C.byref(err))
        dev_err = C.c_uint()
        L.call("ps_fetcher_device_error", self.fetcher, C.byref(dev_err))
        return {"experts_copied": n.value, "bytes_copied": b.value, "host_error": err.value,
                "device_timeout_seq": dev_err.value}

    # --------------------------------------------------------------- helpers
    def _wait(self, ev) -> None:
        if isinstance(ev, tuple):            # striped piece: own stripe + helpers' stripes
            ev, seq = ev
            L.call("ps_stream_wait_event", self.cs, ev)
            self.ring.striper.wait(seq, self.cs)
            return
        L.call("ps_stream_wait_event", self.cs, ev)

    def _sm_count(self) -> int:
        if not hasattr(self, "_sms"):
            self._sms = int(L.device_info().get("sm_count", 148) or 148)
        return self._sms

    def _record(self, stream: int) -> int:
        ev = self.events.next()
        L.call("ps_event_record", ev, stream)
        return ev

    def _pieces(self, sid: int, names: list, even: set, chunk: int | None = None) -> list:
        """Row-aligned pieces (<= chunk bytes) covering `names` in blob order:
        [(byte_start, byte_end, [(tensor, r0, r1), ...])]; 1-row tensors
        (norm vectors) ride in the piece that follows them."""
        chunk = chunk or self.chunk
        blob = self.w.layout.blobs[sid]
        out, items, start, end, big = [], [], None, 0, False
        for name in names:
            t = blob.tensors[name]
            row_b = t.cols * 2
            step = max(1, chunk // row_b)
            if name in even:
                step = max(2, step // 2 * 2)
            r = 0
            while r < t.rows:
                r1 = min(t.rows, r + step)
                b0, b1 = t.offset + r * row_b, t.offset + r1 * row_b
                if big and t.rows > 1 and b1 - start > chunk:
                    out.append((start, end, items))
                    items, start, big = [], None, False
                if start is None:
                    start = b0
                items.append((name, r, r1))
                big = big or t.rows > 1
                end = b1
                r = r1
        if items:
            out.append((start, end, items))
        return out

    def _pieces_hx(self, sid: int, names: list, chunk: int | None = None) -> list:
        """`_pieces` over the shard's hx layout: a matrix splits only between its 64-row
        blocks (runtime/hxcodec.py), raw tensors (norm vectors) whole."""
        chunk = chunk or self.chunk
        blob = self.w.layout.blobs[sid]
        meta = self.hx.tensors[sid]
        out, items, start, end, big = [], [], None, 0, False
        for name in names:
            t = blob.tensors[name]
            off, m = meta[name]
            if m is None:
                units = [(0, t.rows, off, off + t.rows * t.cols * 2)]
            else:
                nb = len(m.block_off) - 1
                step = max(1, int(chunk * nb // max(1, m.nbytes)))
                units = [(b * 64, min(t.rows, (b + step) * 64), off + int(m.block_off[b]),
                          off + int(m.block_off[min(nb, b + step)])) for b in range(0, nb, step)]
            for r, r1, b0, b1 in units:
                if big and t.rows > 1 and b1 - start > chunk:
                    out.append((start, end, items))
                    items, start, big = [], None, False
                if start is None:
                    start = b0
                items.append((name, r, r1))
                big = big or t.rows > 1
                end = b1
        if items:
            out.append((start, end, items))
        return out

    def _hx_consume(self, sid: int, name: str, m, ptr: int, r0: int, r1: int, fn) -> None:
        """Run consumer `fn` over rows [r0, r1) of hx matrix `m` (r0 on a 64-row block;
        `ptr` = device address of that block): expand to bf16 into the expand buffer in
        runs of whole blocks, one consumer call per run. Stream order keeps each
        expansion behind the previous consumer."""
        from .hxcodec import BLOCK_ROWS
        rows_fit = max(BLOCK_ROWS, (self._expand_bytes() // (m.k * 2)) // BLOCK_ROWS * BLOCK_ROWS)
        rows_fit = min(rows_fit, 999 * BLOCK_ROWS)          # block offsets fit one small upload
        lut = self.hx_lut + self.hx.lut_off[(sid, name)]
        base = int(m.block_off[r0 // BLOCK_ROWS])
        ra = r0
        while ra < r1:
            rb = min(r1, ra + rows_fit)
            ba, bb = ra // BLOCK_ROWS, -(-rb // BLOCK_ROWS)
            first = int(m.block_off[ba])
            self._upload(self.hx_meta, (m.block_off[ba:bb] - first).astype(np.int64))
            L.call("ps_hx_expand", ptr + first - base, self.hx_meta, rb - ra, m.k, lut, self.expand, m.k, self.cs)
            self._traced(name, fn, self.expand, ra, rb)
            ra = rb

    def _pieces_coded(self, sid: int, names: list, even: set, chunk: int | None = None) -> list:
        """`_pieces` over the shard's exponent-coded layout (row bytes 1.5 x cols)."""
        chunk = chunk or self.chunk
        blob = self.w.layout.blobs[sid]
        meta = self.coded.tensors[sid]
        out, items, start, end, big = [], [], None, 0, False
        for name in names:
            t = blob.tensors[name]
            off, row_b = meta[name][0], meta[name][1]
            step = max(1, chunk // row_b)
            if name in even:
                step = max(2, step // 2 * 2)
            r = 0
            while r < t.rows:
                r1 = min(t.rows, r + step)
                b0, b1 = off + r * row_b, off + r1 * row_b
                if big and t.rows > 1 and b1 - start > chunk:
                    out.append((start, end, items))
                    items, start, big = [], None, False
                if start is None:
                    start = b0
                items.append((name, r, r1))
                big = big or t.rows > 1
                end = b1
                r = r1
        if items:
            out.append((start, end, items))
        return out

    def _shard(self, sid: int, consumers: list, T: int) -> None:
        """Make a weight shard's tensors addressable and run its consumers in order.

        Pinned / zero-copy shards expose whole tensors. Streamed shards are
        walked piece by piece through the ring: each piece is waited for
        right before its first consumer and released (sealed) after the last
        consumer that reads any tensor in it."""
        mode, dev = self.residency[sid]
        self._zc_direct = False
        if mode == "zerocopy" and (T > GEMV_CORE_MAX_T or (self.stage_zc and self.stage_small)):
            if T > GEMV_MAX_T or self.stage_zc:
                # one pass over the weights: stage CPU-placed shards through the ring (copy
                # engine, once) instead of re-reading host memory per 8 tokens or per tile
                mode = "stream"
            else:   # no room for a ring: the CUDA-core GEMV reads them zero-copy
                self._zc_direct = True
        blob = self.w.layout.blobs[sid]
        own = {c.tensor: i for i, c in enumerate(consumers) if c.tensor is not None}
        readers: dict = {}
        for i, c in enumerate(consumers):
            if c.tensor is not None:
                readers.setdefault(c.tensor, set()).add(i)
            for r in c.reads:
                readers.setdefault(r, set()).add(i)
        names = [n for n in blob.tensors if n in readers]
        self.ptrs = {}
        ci = 0

        def advance_to(target: int) -> None:
            nonlocal ci
            while ci < target:
                c = consumers[ci]
                if c.tensor is not None:
                    raise SpecError(f"consumer order mismatch at {c.tensor}")
                self._traced("core", c.fn, None, 0, 0)
                done(ci)
                ci += 1

        if mode in ("pinned", "zerocopy"):
            zc_coded = (mode == "zerocopy" and self.coded is not None and sid in self.coded.tensors and
                        getattr(self.coded, "mapped", False) and
                        (self.coded_only or os.environ.get("PS_CODED_ZEROCOPY", "1") != "0"))
            res_coded = mode == "pinned" and self.coded_resident(sid)
            if mode == "pinned" and self.hx_resident(sid):
                meta = self.hx.tensors[sid]

                def done(i):
                    pass
                for name in names:
                    t = blob.tensors[name]
                    off, m = meta[name]
                    self.ptrs[name] = dev + off
                    if name in own:
                        advance_to(own[name])
                        if m is not None:
                            self._hx_consume(sid, name, m, dev + off, 0, t.rows, consumers[ci].fn)
                        else:
                            self._traced(name, consumers[ci].fn, dev + off, 0, t.rows)
                        ci += 1
                advance_to(len(consumers))
                return
            if mode == "pinned":
                base = dev
            elif zc_coded:   # the bulk-copy GEMV reads the coded rows straight from host memory
                base = self.coded.shard_ptr(sid)
            else:
                base = self.w.shard_ptr(sid)
            if zc_coded:
                self._stat.zero_copy_bytes += self.coded.shard_bytes[sid]
            elif mode == "zerocopy":
                self._stat.zero_copy_bytes += blob.nbytes
            coded_rows = zc_coded or res_coded
            if coded_rows:
                meta = self.coded.tensors[sid]
            evens = {c.tensor for c in consumers if c.even_rows}
            live = []

            def done(i):
                pass
            for name in names:
                t = blob.tensors[name]
                off = meta[name][0] if coded_rows else t.offset
                self.ptrs[name] = base + off
                if name in own:
                    advance_to(own[name])
                    if coded_rows and meta[name][2] and T > GEMV_MAX_T:
                        # GEMM pass over a coded-resident matrix: rows expanded to bf16 in
                        # pieces of the expand buffer, one GEMM per piece (stream order
                        # keeps the next expansion behind the previous GEMM)
                        step = max(1, self._expand_bytes() // (t.cols * 2))
                        if name in evens:
                            step = max(2, step & ~1)
                        for r0 in range(0, t.rows, step):
                            r1 = min(t.rows, r0 + step)
                            L.call("ps_expand_coded", base + off + r0 * meta[name][1], meta[name][1],
                                   r1 - r0, t.cols, self.expand, t.cols, self.cs)
                            self._traced(name, consumers[ci].fn, self.expand, r0, r1)
                        ci += 1
                        continue
                    if coded_rows and meta[name][2]:
                        self._coded_call = meta[name][1]
                    try:
                        self._traced(name, consumers[ci].fn, base + off, 0, t.rows)
                    finally:
                        self._coded_call = None
                    ci += 1
            advance_to(len(consumers))
            return

        hxs = (self._hx_stream_on() and sid in self.hx.tensors and self.striper is None and
               sid not in self._piece_override)
        coded = (not hxs and self.coded is not None and sid in self.coded.tensors and self.striper is None and
                 sid not in self._piece_override and
                 (T <= GEMV_MAX_T or (bool(self.expand) and self._coded_prefill())))
        expand = coded and T > GEMV_MAX_T   # GEMM pass: coded piece -> bf16 in VRAM -> tcgen05 GEMM
        evens = {c.tensor for c in consumers if c.even_rows}
        if hxs:
            hmeta = self.hx.tensors[sid]
            pieces = self._pieces_hx(sid, names)
            host = self.hx.shard_ptr(sid)
        elif coded:
            meta = self.coded.tensors[sid]
            # an expanded piece (rows x K bf16) must fit the expand buffer: coded rows are
            # >= 0.75 of their bf16 size, so 0.74 of it in coded bytes always does
            pieces = self._pieces_coded(sid, names, evens,
                                        chunk=int(0.74 * min(self.chunk, self._expand_bytes())) if expand else None)
            host = self.coded.shard_ptr(sid)
        else:
            pieces = self._piece_override.pop(sid, None) or self._pieces(sid, names, evens)
            host = self.w.shard_ptr(sid)
        # A piece is released once nothing enqueued later reads it: matrix rows as
        # soon as their consumer has been enqueued for them ("rows" token), small
        # tensors (norms, q/k norms) when every consumer that reads them is done.
        live: list = []       # [region, pending tokens]

        def discharge(entry, token):
            entry[1].discard(token)
            if not entry[1] and entry in live:
                self.ring.seal(entry[0], [self._record(self.cs)])
                live.remove(entry)

        def done(i):
            for entry in live[:]:
                discharge(entry, i)

        for b0, b1, items in pieces:
            pre = self._prefetched.pop((sid, b0), None)
            if pre is not None:
                region, pdev, arrived = pre
            else:
                region, pdev, arrived = self.ring.upload(host + b0, b1 - b0, f"s{sid}@{b0}")
                self._stat.bytes_streamed += b1 - b0
                self._stat.copies += 1
            pending = set()
            for name, _, _ in items:
                rows_consumer = own.get(name) if blob.tensors[name].rows > 1 else None
                if rows_consumer is not None:
                    pending.add(("rows", name))
                pending |= {i for i in readers[name] if i != rows_consumer}
            entry = [region, pending]
            live.append(entry)
            self._wait(arrived)
            for name, r0, r1 in items:
                t = blob.tensors[name]
                hm = None
                if hxs:
                    o, hm = hmeta[name]
                    ptr = pdev + (o - b0) + (int(hm.block_off[r0 // 64]) if hm is not None else r0 * t.cols * 2)
                elif coded:
                    m = meta[name]
                    ptr = pdev + (m[0] + r0 * m[1] - b0)
                else:
                    ptr = pdev + (t.offset + r0 * t.cols * 2 - b0)
                if r0 == 0:
                    self.ptrs[name] = ptr
                if name in own:
                    advance_to(own[name])
                    if hm is not None:
                        self._hx_consume(sid, name, hm, ptr, r0, r1, consumers[ci].fn)
                        if t.rows > 1:
                            discharge(entry, ("rows", name))
                        if r1 == t.rows:
                            done(ci)
                            ci += 1
                        continue
                    if coded and m[2] and expand:
                        L.call("ps_expand_coded", ptr, m[1], r1 - r0, t.cols, self.expand, t.cols, self.cs)
                        ptr = self.expand
                    elif coded and m[2]:   # the consumer's GEMV reads coded rows (stride m[1] bytes)
                        self._coded_call = m[1]
                    try:
                        self._traced(name, consumers[ci].fn, ptr, r0, r1)
                    finally:
                        self._coded_call = None
                    if t.rows > 1:
                        discharge(entry, ("rows", name))
                    if r1 == t.rows:
                        done(ci)
                        ci += 1
        advance_to(len(consumers))
        for entry in live:
            self.ring.seal(entry[0], [self._record(self.cs)])

    def _traced(self, name, fn, *args) -> None:
        if self.tracer is None:
            fn(*args)
            return
        ev0 = self.tracer.begin(self.cs)
        fn(*args)
        self.tracer.end(name or "?", "compute", ev0, self.cs)

    def attach_tracer(self, tracer) -> None:
        self.tracer = tracer
        if self.ring is not None:
            self.ring.tracer = tracer

    def _moe(self, sid: int, layer: int, T: int, gemv: bool, xn: int, norm) -> None:
        """One MoE expert group: router -> top-k -> routed experts -> weighted sum.

        Pinned groups run in place. A streamed (or CPU-placed) group in a GEMV
        pass (t <= 32) is read zero-copy from the host blob, so only the
        routed experts cross the link; in a GEMM pass every expert is touched,
        and the group streams through the ring in whole-expert pieces, the
        expert kernels running per piece over the experts it holds."""
        moe, d = self.moe, self.d
        E, k, eff = moe.n_experts, moe.top_k, moe.expert_ffn_dim
        P = T * k
        blob = self.w.layout.blobs[sid]
        t_norm = blob.tensors[f"L{layer}.ffn_norm"]
        t_router = blob.tensors[f"L{layer}.router"]
        e0 = blob.tensors[f"L{layer}.e0.wgu"]
        stride = blob.tensors[f"L{layer}.e1.wgu"].offset - e0.offset if E > 1 else blob.nbytes
        down_off = blob.tensors[f"L{layer}.e0.wdown"].offset - e0.offset
        mode, dev = self.residency[sid]
        if mode == "zerocopy" and not gemv:
            mode = "stream"
        elif mode == "stream" and gemv:
            mode = "zerocopy"

        # one token: the k routed experts as row groups of two bulk-copy launches,
        # combine fused, no plan (csrc/moe_decode.cu)
        planned = self.residency[sid][0]
        fetched = gemv and planned == "stream" and bool(self.expert_slots)
        t1 = (gemv and T == 1 and d <= 2048 and eff <= 2048 and (fetched or mode == "pinned") and
              k <= 16 and   # moe_down_t1_kernel: one ring slot per routed expert
              os.environ.get("PS_MOE_DECODE", "1") != "0")

        def route(base):
            norm(base + t_norm.offset)
            # a router read from host memory takes the CUDA-core GEMV (no tensor map over it)
            self._zc_direct = base == self.w.shard_ptr(sid)
            self._matmul(T, xn, base + t_router.offset, E, d, self.m_logits, E, L.PS_EPI_STORE)
            self._zc_direct = False
            L.call("ps_moe_route_topk", self.m_logits, E, T, E, k, 1, self.m_ids, self.m_w, self.cs)
            if not t1:
                L.call("ps_moe_plan", self.m_ids, P, E, self.m_plan, self.cs)

        # routed experts coded through the fetcher (one-token kernels only): hx-coded
        # (expanded to bf16 scratch slots on arrival), else 12-bit (decoded in the kernels)
        cexp = hxe = None
        if t1 and fetched and self._hx_experts_on(1):
            hxe = self.hx.experts.get(sid)
        if (hxe is None and t1 and fetched and self.coded is not None and
                os.environ.get("PS_CODED_EXPERTS", "1") != "0"):
            cexp = getattr(self.coded, "experts", {}).get(sid)

        spec_n = self._spec_n(T) if (t1 and fetched and hxe is not None) else 0

        def hx_gate_up(ebase, slot_map, r0, r1):
            """Routed experts of ranks [r0, r1): spans -> bf16 scratch experts (blob layout),
            then their gate/up + SwiGLU. With speculative prefetch rank r's span is in slot
            m_sor[r] (the fetcher's placement), else in slot r."""
            sc, sst = self.hx_escratch, stride
            span0, sor = (ebase, self.m_sor + r0 * 4) if spec_n else (ebase + r0 * sb, None)
            L.call("ps_hx_expand_experts2", span0, sb, sor, r1 - r0,
                   0, hxe["gu_off"], hxe["gu_rows"], hxe["gu_k"], self.hx_lut + self.hx.lut_off[(sid, "wgu")], 0,
                   hxe["nb_gu"], hxe["dn_off"], hxe["dn_rows"], hxe["dn_k"],
                   self.hx_lut + self.hx.lut_off[(sid, "wdown")], down_off, sc + r0 * sst, sst, self.cs)
            L.call("ps_moe_decode_experts_phase", xn, self.m_ids, k, slot_map, sc, sst, 0, down_off, eff, d,
                   self.m_h, self.m_w, self.x, 1, r0, r1, self.cs)

        def decode_t1(ebase, slot_map):
            if hxe is not None:   # (unsplit: every rank has landed)
                hx_gate_up(ebase, slot_map, 0, k)
                L.call("ps_moe_decode_experts_phase", xn, self.m_ids, k, slot_map, self.hx_escratch, stride, 0,
                       down_off, eff, d, self.m_h, self.m_w, self.x, 2, 0, k, self.cs)
                return
            if cexp is not None:
                L.call("ps_moe_decode_experts_c", xn, self.m_ids, k, slot_map, ebase, sb, 0, cexp[2], eff, d,
                       cexp[4], cexp[5], self.m_h, self.m_w, self.x, self.cs)
                return
            L.call("ps_moe_decode_experts", xn, self.m_ids, k, slot_map, ebase, stride if not slot_map else sb,
                   0, down_off, eff, d, self.m_h, self.m_w, self.x, self.cs)

        def experts(ebase, lo, hi):
            L.call("ps_moe_expert_gu", xn, d, 0 if gemv else 1, self.m_plan, E, P, k, ebase, stride, 0,
                   eff, d, self.m_h, lo, hi, self.cs)
            L.call("ps_moe_expert_down", self.m_h, self.m_plan, E, P, ebase, stride, down_off, eff, d,
                   self.m_out, lo, hi, self.cs)

        if fetched:
            # routed experts through the copy engine (csrc/fetcher.cu)
            host = self.w.shard_ptr(sid)
            _, _, _, ebytes = self._expert_geometry(sid, layer)
            slots, sb = self.expert_slots, self.expert_slot_bytes
            src0, src_stride = host + e0.offset, stride
            if hxe is not None:       # hx experts: ~35 % fewer bytes per routed expert
                src0, src_stride, ebytes = self.hx.shard_ptr(sid), hxe["stride"], hxe["stride"]
            elif cexp is not None:    # coded experts: 25 % fewer bytes per routed expert
                src0, src_stride, ebytes = self.coded.shard_ptr(sid) + cexp[0], cexp[1], cexp[3]
            # PS_MOE_SPLIT=1: hx experts arrive in two halves, the first half's expansion and
            # gate/up running while the second half is still crossing the link (flag seq - 1,
            # then seq). Measured neutral on config 3 (19.85 vs 19.80 tokens/s): the chain
            # after the last expert lands is the expansion's fixed latency (one 256-weight
            # serial decode), the same for 4 experts as for 8. Off by default.
            split = k // 2 if (hxe is not None and k >= 2 and not spec_n and
                               os.environ.get("PS_MOE_SPLIT", "0") == "1") else 0
            self.fetch_seq = (self.fetch_seq + (2 if split else 1)) & 0xFFFFFFFF
            if self.fetch_seq < 2:
                self.fetch_seq = 2
            seq = self.fetch_seq
            pre = self._prefix_dev.pop(sid, None)     # ffn_norm + router staged by gap filling
            if pre is not None:
                region, base, arrived = pre
                self._wait(arrived)
            else:
                base = host
                self._stat.zero_copy_bytes += e0.offset
            self._traced(f"L{layer}.router+topk", route, base)
            if pre is not None:
                self.ring.seal(region, [self._record(self.cs)])
            # speculative prefetch: this layer's hits sit in prediction set `set_cur`; the
            # next layer's router (staged by gap filling) picks spec_n experts from this
            # layer's post-attention state, copied into set `set_next` behind this layer's
            # experts (csrc/fetcher.cu)
            set_cur = set_next = -1
            nxt_hx = None
            if spec_n:
                pend = self._spec_pending
                set_cur = pend[1] if pend is not None and pend[0] == layer else -1
                self._spec_pending = None
                nxt = self.by_layer_kind.get((layer + 1, ShardKind.MOE_EXPERT_GROUP))
                pre_n = self._prefix_dev.get(nxt.id) if nxt is not None else None
                nxt_hx = self.hx.experts.get(nxt.id) if pre_n is not None else None
                if nxt_hx is not None:
                    set_next = 1 - set_cur if set_cur >= 0 else 0
                    nblob = self.w.layout.blobs[nxt.id]
                    _, nbase, narrived = pre_n
                    self._wait(narrived)

                    def predict(_p, _a, _b):
                        L.call("ps_rmsnorm", self.x, d, 0, T, nbase + nblob.tensors[f"L{layer + 1}.ffn_norm"].offset,
                               d, self.arch.rms_eps, self.m_xp, d, 0, self.cs)
                        self._matmul(T, self.m_xp, nbase + nblob.tensors[f"L{layer + 1}.router"].offset, E, d,
                                     self.m_logits, E, L.PS_EPI_STORE)
                        L.call("ps_moe_route_topk", self.m_logits, E, T, E, spec_n, 1, self.m_pids, self.m_pw,
                               self.cs)
                    self._traced(f"L{layer}.predict L{layer + 1}", predict, 0, 0, 0)
                    self._spec_pending = (layer + 1, set_next)

            def fetch(_p, _a, _b):
                if spec_n:
                    L.call("ps_fetcher_submit_spec", self.fetcher, seq, src0, src_stride, ebytes, slots, sb,
                           self.expert_slot_count, self.hx.shard_ptr(nxt.id) if nxt_hx else None,
                           nxt_hx["stride"] if nxt_hx else 0, nxt_hx["stride"] if nxt_hx else 0)
                    L.call("ps_moe_publish_spec", self.fetcher, self.m_ids, P, E, self.m_slotmap, seq,
                           self.m_pids, spec_n, self.m_spec, set_cur, set_next, P, self.m_sor, self.cs)
                    L.call("ps_wait_flag", self.fetcher, seq, self.cs)
                    return
                if split:
                    L.call("ps_fetcher_submit_split", self.fetcher, seq, src0, src_stride, ebytes, slots, sb, split)
                else:
                    L.call("ps_fetcher_submit", self.fetcher, seq, src0, src_stride, ebytes, slots, sb)
                L.call("ps_moe_publish", self.fetcher, self.m_ids, P, E, self.m_slotmap, seq, self.cs)
                L.call("ps_wait_flag", self.fetcher, seq - 1 if split else seq, self.cs)
                if os.environ.get("PS_FETCH_DEBUG"):
                    self._fetch_debug(layer, seq, P, E, src0, src_stride, ebytes, slots, sb)

            def run(_p, _a, _b):
                if t1 and split:
                    hx_gate_up(slots, self.m_slotmap, 0, split)           # first half, landed
                    L.call("ps_wait_flag", self.fetcher, seq, self.cs)     # the rest
                    hx_gate_up(slots, self.m_slotmap, split, k)
                    L.call("ps_moe_decode_experts_phase", xn, self.m_ids, k, self.m_slotmap, self.hx_escratch,
                           stride, 0, down_off, eff, d, self.m_h, self.m_w, self.x, 2, 0, k, self.cs)
                    return
                if t1:
                    decode_t1(slots, self.m_slotmap)
                    return
                L.call("ps_moe_expert_gu_mapped", xn, d, 0, self.m_plan, E, P, k, slots, sb, 0, eff, d,
                       self.m_h, 0, E, self.m_slotmap, self.cs)
                L.call("ps_moe_expert_down_mapped", self.m_h, self.m_plan, E, P, slots, sb, down_off, eff, d,
                       self.m_out, 0, E, self.m_slotmap, self.cs)

            self._throttle_host()
            self._traced(f"L{layer}.experts fetch", fetch, 0, 0, 0)
            self._gapfill_step()      # the copy stream may move the next prefix / head piece now
            self._traced(f"L{layer}.experts", run, 0, 0, 0)
            self._stat.bytes_streamed += min(E, P) * ebytes
            self._stat.copies += min(E, P)
            if spec_n:   # the fetcher decides what crosses the link: settled after the pass
                self._stat.fetch_seqs.append((seq, min(E, P) * ebytes, ebytes,
                                              spec_n * nxt_hx["stride"] if set_next >= 0 else 0,
                                              min(E, P) if set_cur >= 0 else 0, spec_n if set_next >= 0 else 0))
            if not t1:
                L.call("ps_moe_combine", self.m_out, self.m_plan, E, P, self.m_w, T, k, d, self.x, d, self.cs)
            return

        if mode == "pinned" and t1:
            self._traced(f"L{layer}.router+topk", route, dev)
            self._traced(f"L{layer}.experts", lambda *_: decode_t1(dev + e0.offset, None), 0, 0, 0)
            return
        if mode in ("pinned", "zerocopy"):
            base = dev if mode == "pinned" else self.w.shard_ptr(sid)
            self._traced(f"L{layer}.router+topk", route, base)
            self._traced(f"L{layer}.experts", experts, base + e0.offset, 0, E)
            if mode == "zerocopy":
                touched = min(E, P)
                self._stat.zero_copy_bytes += e0.offset + touched * stride
                self._gapfill_step()
        elif self._hx_prefill_experts(sid):
            # GEMM pass over a streamed group, hx-coded (~0.65 x the bf16 bytes): the bf16
            # prefix (ffn_norm + router) first, then pieces of whole hx expert spans; each
            # piece is expanded a few experts at a time into the expansion buffer (blob
            # layout) and the expert kernels run on those experts, bit-identical to bf16
            hxg = self.hx.experts[sid]
            host, hs = self.w.shard_ptr(sid), hxg["stride"]
            region, pdev, arrived = self.ring.upload(host, e0.offset, f"moe{sid} prefix")
            self._stat.bytes_streamed += e0.offset
            self._stat.copies += 1
            self._wait(arrived)
            self._traced(f"L{layer}.router+topk", route, pdev)
            self.ring.seal(region, [self._record(self.cs)])
            hx_base = self.hx.shard_ptr(sid)
            lut_gu = self.hx_lut + self.hx.lut_off[(sid, "wgu")]
            lut_dn = self.hx_lut + self.hx.lut_off[(sid, "wdown")]
            per_piece = max(1, self.chunk // hs)
            per_run = max(1, self._expand_bytes() // stride)

            def expand_run(sp, a, b):
                L.call("ps_hx_expand_experts2", sp, hs, None, b - a,
                       0, hxg["gu_off"], hxg["gu_rows"], hxg["gu_k"], lut_gu, 0,
                       hxg["nb_gu"], hxg["dn_off"], hxg["dn_rows"], hxg["dn_k"], lut_dn, down_off,
                       self.expand, stride, self.cs)
                experts(self.expand - a * stride, a, b)    # expert e at expand + (e - a) * stride

            for lo in range(0, E, per_piece):
                hi = min(E, lo + per_piece)
                region, pdev, arrived = self.ring.upload(hx_base + lo * hs, (hi - lo) * hs, f"moe{sid}hx@{lo}")
                self._stat.bytes_streamed += (hi - lo) * hs
                self._stat.copies += 1
                self._wait(arrived)
                for a in range(lo, hi, per_run):
                    b = min(hi, a + per_run)
                    self._traced(f"L{layer}.experts[{a}:{b})", expand_run, pdev + (a - lo) * hs, a, b)
                self.ring.seal(region, [self._record(self.cs)])
        else:
            host = self.w.shard_ptr(sid)
            per_piece = max(1, (self.chunk - e0.offset) // stride)
            lo = 0
            first = True
            while lo < E:
                hi = min(E, lo + (per_piece if not first else max(1, per_piece)))
                b0 = 0 if first else e0.offset + lo * stride
                b1 = e0.offset + hi * stride
                region, pdev, arrived = self.ring.upload(host + b0, b1 - b0, f"moe{sid}@{lo}")
                self._stat.bytes_streamed += b1 - b0
                self._stat.copies += 1
                self._wait(arrived)
                if first:
                    self._traced(f"L{layer}.router+topk", route, pdev)
                self._traced(f"L{layer}.experts[{lo}:{hi})", experts, pdev + e0.offset - b0, lo, hi)
                self.ring.seal(region, [self._record(self.cs)])
                first = False
                lo = hi
        L.call("ps_moe_combine", self.m_out, self.m_plan, E, P, self.m_w, T, k, d, self.x, d, self.cs)

    # ------------------------------------------------- gap filling (MoE decode)
    def _plan_gapfill(self, gemv: bool, R: int, T: int = 0) -> None:
        """Zero-copy / fetched MoE decode leaves the host link idle between layers
        (expert kernels, the next layer's attention, router and top-k run while no
        expert byte can move yet). Two kinds of bytes are known in advance and fill
        those gaps, uploaded on the ring's copy stream gated on the cs event that
        marks "this layer's experts are in VRAM" (fetched) or "this layer's experts
        ran" (zero-copy):
        * the next fetched MoE layer's prefix (ffn_norm + router, ~0.5 MB), so its
          route runs from VRAM instead of reading the router over PCIe;
        * one piece of the output head — the pass's one ring-streamed dense shard,
          read only at its end — per MoE layer.
        Enabled only when nothing else in the pass uses the ring."""
        self._gapfill, self._piece_override, self._prefetched = None, {}, {}
        self._prefix_queue, self._prefix_dev = [], {}
        self._spec_pending = None
        if not (gemv and R and self.moe is not None and self.ring is not None) or \
                os.environ.get("PS_GAPFILL", "1") == "0":
            return
        head_sid = self.by_layer_kind[(self.spec.n_layers, ShardKind.OUTPUT_HEAD)].id
        head_streams = self.residency[head_sid][0] == "stream"   # a spare-pinned head needs no pieces
        moe_streamed = []
        for sid, (mode, _) in self.residency.items():
            kind = self.shard_kind[sid]
            if kind is ShardKind.MOE_EXPERT_GROUP:
                if mode in ("zerocopy", "stream"):
                    moe_streamed.append(sid)
            elif sid != head_sid and mode == "stream":
                return
        zc = len(moe_streamed)
        if zc == 0 or any(m == "stream" for m in self.kv_mode.values()):
            return
        pieces = []
        if head_streams:
            blob = self.w.layout.blobs[head_sid]
            names = [n for n in blob.tensors if n in ("final_norm", "lm_head")]
            chunk = max(4 << 20, -(-blob.nbytes // zc))
            pieces = self._pieces(head_sid, names, set(), chunk=min(chunk, self.chunk))
            if sum((b1 - b0 + 255) // 256 * 256 for b0, b1, _ in pieces) > self.ring.capacity * 8 // 10:
                return
            self._piece_override[head_sid] = pieces
        self._gapfill = (head_sid, list(pieces))
        # router prefixes of the fetched MoE layers, in layer order; the first goes up now
        if self.expert_slots:
            fetched = sorted((self.shards[sid].layer_index, sid) for sid in moe_streamed
                             if self.residency[sid][0] == "stream")
            self._prefix_queue = [sid for _, sid in fetched]
            self._upload_prefix()
            if self._spec_n(T):   # two ahead: the next layer's router predicts its experts
                self._upload_prefix()
        # the pass opens with pinned layers and the first routing chain before any
        # expert byte can move: two head pieces keep the link busy meanwhile
        for _ in range(min(2, len(pieces))):
            self._upload_head_piece()

    def _upload_prefix(self) -> None:
        if not self._prefix_queue:
            return
        sid = self._prefix_queue.pop(0)
        layer = self.shards[sid].layer_index
        e0_off = self._expert_geometry(sid, layer)[0]
        self._prefix_dev[sid] = self.ring.upload(self.w.shard_ptr(sid), e0_off, f"moe{sid} prefix")
        self._stat.bytes_streamed += e0_off
        self._stat.copies += 1

    def _gapfill_step(self) -> None:
        """Called right after a MoE layer's experts are available (fetched: after the
        wait kernel) or consumed (zero-copy): the copy stream uploads the next MoE
        prefix and the next head piece once the compute stream reaches this point."""
        if not self._gapfill:
            return
        sid, todo = self._gapfill
        if not todo and not self._prefix_queue:
            return
        L.call("ps_stream_wait_event", self.h2d, self._record(self.cs))
        self._upload_prefix()
        self._upload_head_piece()

    def _upload_head_piece(self) -> None:
        sid, todo = self._gapfill
        if not todo:
            return
        b0, b1, _ = todo.pop(0)
        self._prefetched[(sid, b0)] = self.ring.upload(self.w.shard_ptr(sid) + b0, b1 - b0, f"s{sid}@{b0}")
        self._stat.bytes_streamed += b1 - b0
        self._stat.copies += 1

    def _matmul(self, T, act, W, N, K, out, ldo, epi) -> None:
        """out (epi)= act @ W[:N]^T for T tokens: GEMV on fp32 act (T <= 32)
        or the tcgen05 GEMM on bf16 act."""
        coded = self._coded_call
        if T > GEMV_MAX_T:
            L.call("ps_gemm_bf16", act, T, K, K, W, N, K, out, ldo, epi, self.cs)
        elif T > GEMV_CORE_MAX_T and not self._zc_direct:   # one pass over W for the batch (tcgen05)
            L.call("ps_gemv_tc", act, K, T, W, N, K, coded if coded is not None else K,
                   1 if coded is not None else 0, out, ldo, epi, self.tcws, self._tcws_bytes, self.cs)
        elif coded is not None:   # t <= 8 per launch (zero-copy rows at 9..32 tokens: chunks of 8)
            for t0 in range(0, T, GEMV_CORE_MAX_T):
                L.call("ps_gemv_bf16c", act + t0 * K * 4, K, min(GEMV_CORE_MAX_T, T - t0), W, N, K, coded,
                       out + t0 * ldo * 4, ldo, epi, self.cs)
        else:
            L.call("ps_gemv_bf16", act, K, T, W, N, K, K, out, ldo, epi, self.cs)

    def _upload(self, dst: int, arr: np.ndarray) -> None:
        arr = np.ascontiguousarray(arr, dtype=np.int32)
        if arr.nbytes == 0:
            return
        if arr.nbytes <= 4000:
            L.call("ps_upload_small", dst, arr.ctypes.data, arr.nbytes, self.cs)
        else:
            self._h2d_sync(dst, arr)

    # ----------------------------------------------------------------- the pass
    def _pdl_ok(self, T: int) -> bool:
        """Programmatic dependent launch for this pass (csrc/common.cuh): only when every
        weight it reads is VRAM-resident or host-mapped (no ring copies, no fetched
        experts, no stripes), so the only producers of a kernel's inputs are earlier
        kernels on the compute stream."""
        if (T > GEMV_MAX_T or os.environ.get("PS_PDL", "1") == "0" or self.striper is not None
                or (self.stage_zc and self.stage_small)):
            return False
        if os.environ.get("PS_PDL_STREAMED", "0") == "1":   # experiment: ring + fetcher passes too
            return True
        return (not self.expert_slots and
                all(m != "stream" for m, _ in self.residency.values()) and
                all(m != "stream" for m in self.kv_mode.values()))

    def run_pass(self, ps: PassSpec) -> PassStats:
        pdl = self._pdl_ok(ps.T)
        if pdl:
            L.call("ps_set_pdl", 1)
        try:
            return self._run_pass(ps)
        finally:
            if pdl:
                L.call("ps_set_pdl", 0)

    def _run_pass(self, ps: PassSpec) -> PassStats:
        T = ps.T
        if T > self.T_tier:
            raise SpecError(f"pass of {T} tokens exceeds the tier's {self.T_tier}-token buffers")
        nb = len(ps.slots)
        self.settle()
        self._stat = PassStats(self.tier, T)
        calls0 = L.counters["kernel_calls"]
        gemv = T <= GEMV_MAX_T
        d, hq = self.d, self.h * self.hd

        pos = np.empty(T, np.int32)
        req = np.empty(T, np.int32)
        q_start = np.zeros(nb + 1, np.int32)
        k = 0
        for j, (slot, n, p0) in enumerate(zip(ps.slots, ps.n_new, ps.p0)):
            pos[k:k + n] = np.arange(p0, p0 + n, dtype=np.int32)
            req[k:k + n] = slot
            k += n
            q_start[j + 1] = k
        lens = np.array([p0 + n for p0, n in zip(ps.p0, ps.n_new)], np.int32)
        if int(lens.max()) > self.cap:
            raise SpecError(f"context {int(lens.max())} exceeds the planned {self.cap}")
        p0a = np.array(ps.p0, np.int32)
        rows = np.array([int(q_start[j + 1]) - 1 for j in ps.sample], np.int32)
        self._upload(self.i_pos, pos)
        self._upload(self.i_req, req)
        self._upload(self.i_meta, np.concatenate([q_start, p0a, lens,
                                                  np.array(ps.slots, np.int32)]))
        self._upload(self.i_rows, rows)
        i_qstart = self.i_meta
        i_p0 = i_qstart + 4 * (nb + 1)
        i_lens = i_p0 + 4 * nb
        i_slot = i_lens + 4 * nb
        max_len, max_new = int(lens.max()), int(max(ps.n_new))
        # paged KV: pages for every new position, then the pages a streamed cache needs
        # in the ring (existing rows the attention reads) and writes back (new rows)
        for slot, n, p0 in zip(ps.slots, ps.n_new, ps.p0):
            self.kv_pages.ensure(slot, p0 + n)
        self._sync_block_table()
        kv_read = KvPagePool.runs(pg for slot, p0 in zip(ps.slots, ps.p0)
                                  for pg in self.kv_pages.pages(slot, 0, p0))
        kv_write = KvPagePool.runs(pg for slot, n, p0 in zip(ps.slots, ps.n_new, ps.p0)
                                   for pg in self.kv_pages.pages(slot, p0, p0 + n))
        kv_span = 1 + max(p + c - 1 for p, c in kv_read + kv_write)   # ring window, in pages
        use_decode_kernel = ps.decode_only and gemv

        if ps.ids is not None:
            self._upload(self.i_ids, np.asarray(ps.ids, np.int32))
            ids_ptr = self.i_ids
        else:
            if self._prev_sample_slots != list(ps.slots):
                raise SpecError("a pass without ids must follow a pass that sampled the same slots")
            ids_ptr = self.i_tok          # the previous sampling pass's slot
        L.call("ps_embed_gather", self.w.embed, ids_ptr, T, d, self.x, d, self.cs)
        early = self._early_head_plan(T, len(ps.sample))
        if early is not None:
            self.head_seq = (self.head_seq + 1) & 0x7FFFFFFF or 1
            if self._head_free is not None:   # the previous pass's argmax has read the logits
                L.call("ps_stream_wait_event", self.hs, self._head_free)
            cap = max(1, self._sm_count() // 2)
            L.call("ps_gemv_head_early", self.xs, d, early[1], self.V, early[2], early[3], self.logits, cap,
                   self.head_flag, self.head_seq, self.hs)
            L.call("ps_event_record", self._ev_head_done, self.hs)
            self._stat.zero_copy_bytes += early[4]

        xn = self.xn32 if gemv else self.xn16
        att = self.att32 if gemv else self.att16
        hid = self.hid32 if gemv else self.hid16
        esz = 4 if gemv else 2
        scale = 1.0 / math.sqrt(self.hd)
        eps = self.arch.rms_eps
        bt, pps, page = self.i_bt, self.pps, KV_PAGE_ROWS

        def norm(w_ptr):
            L.call("ps_rmsnorm", self.x, d, 0, T, w_ptr, d, eps, xn, d, 0 if gemv else 1, self.cs)

        self._plan_gapfill(gemv, len(ps.sample), T)

        for layer in range(self.spec.n_layers):
            attn_sid = self.by_layer_kind[(layer, ShardKind.ATTENTION)].id
            ffn_sid = self.by_layer_kind[(layer, ShardKind.FFN if self.moe is None
                                          else ShardKind.MOE_EXPERT_GROUP)].id
            # ---- KV_i, hoisted before Attn_i
            mode = self.kv_mode[layer]
            kv_region = None
            kv_pool_pages = self.kv_pages.n_pages
            if mode == "pinned":
                kv_base = self.kv_vram[layer]
            elif mode == "zerocopy" and gemv:
                kv_base = self._kv_host_ptr(layer)
            else:
                # a window of the layer's host pool in the ring, pages at their pool
                # offsets: the pages holding rows the attention reads come up; pages that
                # only receive new rows need room, not bytes
                wb = self.kv_writeback.get(layer)
                if wb is not None and kv_read:
                    # the host home must hold the previous pass's appended rows
                    L.call("ps_stream_wait_event", self.h2d, wb)
                kv_region, kv_base, arrived = self.ring.upload_runs(
                    self._kv_host_ptr(layer), [(p * self.page_bytes, c * self.page_bytes) for p, c in kv_read],
                    kv_span * self.page_bytes, f"kv{layer}")
                kv_pool_pages = kv_span
                up = sum(c for _, c in kv_read) * self.page_bytes
                self._stat.bytes_streamed += up
                self._stat.kv_bytes += up
                self._stat.copies += len(kv_read)
                self._wait(arrived)

            # ---- Attn_i
            def core(_p, _a, _b, layer=layer, kv_base=kv_base, kv_region=kv_region, kv_pool_pages=kv_pool_pages):
                qn = self.ptrs.get(f"L{layer}.q_norm", 0)
                kn = self.ptrs.get(f"L{layer}.k_norm", 0)
                L.call("ps_qkv_rope_append", self.qkv, self.qkv_rows, T, self.h, self.kv, self.hd,
                       self.i_pos, self.i_req, kv_base, self.row_elems, bt, pps, page, self.rope,
                       qn, kn, eps, self.cs)
                if use_decode_kernel:
                    L.call("ps_attn_decode", self.qkv, self.qkv_rows, nb, self.h, self.kv, self.hd,
                           i_slot, kv_base, self.row_elems, bt, pps, page, i_lens, max_len, scale,
                           att, hq, self.ws, self.ws_floats, self.cs)
                else:
                    # tcgen05 / TMEM / TMA flash attention over the pages (attention_tc.cu)
                    L.call("ps_attn_prefill_tc", self.qkv, self.qkv_rows, nb, i_qstart, i_p0, i_slot,
                           max_new, self.h, self.kv, self.hd, kv_base, self.row_elems, bt, pps, page,
                           kv_pool_pages, scale, att, hq, 0 if gemv else 1, self.cs)
                if kv_region is not None:
                    # pages with appended rows -> the layer's host home (D2H stream), then release
                    L.call("ps_stream_wait_event", self.d2h, self._record(self.cs))
                    ev0 = self.tracer.begin(self.d2h) if self.tracer else None
                    n = self._copy_pages(self._kv_host_ptr(layer), kv_base, kv_write, self.d2h)
                    if ev0 is not None:
                        self.tracer.end(f"kv{layer} write-back", "d2h", ev0, self.d2h)
                    self._stat.kv_writeback_bytes += n
                    wb = self._record(self.d2h)
                    self.kv_writeback[layer] = wb
                    self.ring.seal(kv_region, [wb])

            reads = (f"L{layer}.q_norm", f"L{layer}.k_norm") if self.arch.qk_norm else ()
            self._shard(attn_sid, [
                Consumer(f"L{layer}.attn_norm", lambda p, a, b: norm(p)),
                Consumer(f"L{layer}.wqkv", lambda p, r0, r1: self._matmul(
                    T, xn, p, r1 - r0, d, self.qkv + r0 * 4, self.qkv_rows, L.PS_EPI_STORE)),
                Consumer(None, core, reads=reads),
                Consumer(f"L{layer}.wo", lambda p, r0, r1: self._matmul(
                    T, att, p, r1 - r0, hq, self.x + r0 * 4, d, L.PS_EPI_ACCUM)),
            ], T)

            # ---- FFN_i or MoE_i
            if self.moe is not None:
                self._moe(ffn_sid, layer, T, gemv, xn, norm)
                continue
            self._shard(ffn_sid, [
                Consumer(f"L{layer}.ffn_norm", lambda p, a, b: norm(p)),
                Consumer(f"L{layer}.wgu", lambda p, r0, r1: self._matmul(
                    T, xn, p, r1 - r0, d, hid + (r0 // 2) * esz, self.ffn, L.PS_EPI_SWIGLU),
                    even_rows=True),
                Consumer(f"L{layer}.wdown", lambda p, r0, r1: self._matmul(
                    T, hid, p, r1 - r0, self.ffn, self.x + r0 * 4, d, L.PS_EPI_ACCUM)),
            ], T)

        # ---- head, on the sampled rows only (HEAD_ROWS_CAP, model_graph.py:30-33)
        R = len(ps.sample)
        if R:
            head_sid = self.by_layer_kind[(self.spec.n_layers, ShardKind.OUTPUT_HEAD)].id

            def hnorm(p, a, b):
                L.call("ps_rmsnorm", self.x, d, self.i_rows, R, p, d, eps, self.xs, d, 0, self.cs)

            def lm(p, r0, r1):
                self._matmul(R, self.xs, p, r1 - r0, d, self.logits + r0 * 4, self.V, L.PS_EPI_STORE)

            self.tok_slot = (self.tok_slot + 1) % 8
            self.i_tok = self.i_tok_ring + self.tok_slot * self.B * 4

            def greedy(p, a, b):
                L.call("ps_argmax", self.logits, R, self.V, self.V, self.i_tok, self.cs)

            if early is not None:
                hnorm(early[0], 0, 1)                                       # x final ...
                L.call("ps_set_flag", self.head_flag, self.head_seq, self.cs)   # ... says so
                L.call("ps_stream_wait_event", self.cs, self._ev_head_done)
                # a plain launch after the event wait: the argmax's programmatic dependency
                # is on a kernel that itself started after the head GEMV finished
                L.call("ps_set_flag", self.head_flag, self.head_seq, self.cs)
                greedy(None, 0, 0)
                L.call("ps_event_record", self._ev_head_free, self.cs)
                self._head_free = self._ev_head_free
            else:
                self._shard(head_sid, [Consumer("final_norm", hnorm), Consumer("lm_head", lm),
                                       Consumer(None, greedy)], R)
            L.call("ps_stream_wait_event", self.d2h, self._record(self.cs))
            dst = self.host_tok + (self.host_tok_i % 4096) * self.B * 4
            self.host_tok_i += 1
            L.memcpy_async(dst, self.i_tok, R * 4, self.d2h)
            sampled = [ps.slots[j] for j in ps.sample]
            ev = self.tok_events[self.host_tok_i % len(self.tok_events)]
            L.call("ps_event_record", ev, self.d2h)
            self.host_tokens.append((dst, R, ev, sampled))
            self._prev_sample_slots = sampled
        for slot, n, p0 in zip(ps.slots, ps.n_new, ps.p0):
            self.kv_len[slot] = max(self.kv_len[slot], p0 + n)
        self._stat.kernel_calls = L.counters["kernel_calls"] - calls0
        self.stats.append(self._stat)
        if self._stat.fetch_seqs:
            self._unsettled.append(self._stat)
        return self._stat

    # ------------------------------------------------------------------ results
    def collect_tokens(self) -> list:
        """Wait for and return [(slots, tokens)] of every sampling pass so far."""
        out = []
        for dst, R, ev, slots in self.host_tokens:
            L.call("ps_event_synchronize", ev)
            out.append((slots, np.ctypeslib.as_array((C.c_int32 * R).from_address(dst)).copy()))
        self.host_tokens = []
        return out

    def logits_host(self, rows: int) -> np.ndarray:
        """fp32 logits of the last sampling pass (synchronises)."""
        self.synchronize()
        import torch
        t = self.arena.tensor(self.logits, rows * self.V * 4).view(torch.float32)
        return t.reshape(rows, self.V).cpu().numpy()

    def check_errors(self) -> None:
        """Raise if any device-side wait gave up or the fetcher failed: a timed-out
        wait lets its kernel finish on stale ring / slot bytes, so the pass's tokens
        are invalid. Host-mapped fault words (a plain load, no synchronisation), plus
        the fetcher's host-side error code."""
        L.raise_on_fault()
        if self.fetcher is not None:
            err = C.c_int()
            L.call("ps_fetcher_info", self.fetcher, None, None, None, None, C.byref(err))
            if err.value:
                raise L.DeviceFault(f"expert fetcher host error {err.value} "
                                    "(1: routing never published, 2: bad expert id, 3: copy failed)")

    def synchronize(self) -> None:
        for s in (self.cs, self.h2d, self.d2h, self.hs):
            L.call("ps_stream_synchronize", s)
        self.settle()

    def settle(self) -> None:
        """Replace the link bytes counted for speculatively fetched layers (k experts each)
        by what the fetcher copied (misses + predictions), for every job the fetcher has
        processed (all of them after a synchronize). Also called at each pass start, so the
        fetcher's per-seq record (a ring of 65536 seqs) is read long before it wraps."""
        if self.fetcher is None or not self._unsettled:
            return
        keep = []
        for st in self._unsettled:
            rest = []
            for job in st.fetch_seqs:
                seq, counted, ebytes, pred_bytes, routed, npred = job
                got = C.c_longlong(-1)
                L.call("ps_fetcher_seq_bytes", self.fetcher, seq, C.byref(got))
                if got.value < 0:
                    rest.append(job)
                    continue
                st.bytes_streamed += got.value - counted
                st.spec_predicted += npred
                st.spec_pred_bytes += pred_bytes
                misses = (got.value - pred_bytes) // max(1, ebytes)
                if routed:   # the routed experts that were not copied were prefetched hits
                    st.spec_routed += routed
                    st.spec_hits += routed - misses
            st.fetch_seqs = rest
            if rest:
                keep.append(st)
        self._unsettled = keep

    def close(self) -> None:
        if self.fetcher is not None:
            self.synchronize()
            L.call("ps_fetcher_destroy", self.fetcher)
            self.fetcher = None
        if self.kv_host:
            self.synchronize()
            L.host_free(self.kv_host)
            L.host_free(self.host_stage)
            L.host_free(self.host_tok)
            self.kv_host = 0
