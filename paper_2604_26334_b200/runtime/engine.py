"""User-facing engine: model load, VRAM budget, plan, prefill / decode / generate.

This is the drop-in for the reference's inference path. Planning is the
reference-compatible planner (`paper_2604_26334_b200.planning`, bit-exact
with `pkg/src/shardplan/planner.py`); the loop is `simulate_inference`'s
(`pkg/src/shardplan/simulator.py:239-314`) — same tier pick, same chunked
prefill, same definitions of TTFT, decode TPS and E2EL — but every pass is
a real GPU pass of `Executor.run_pass` instead of `simulate_schedule`.

    eng = Engine("llama3.1-8b", budget_bytes=4e9, context_len=2304)
    out = eng.generate([prompt_ids], gen_len=256)
    out.tokens, out.ttft_s, out.tps
"""

from __future__ import annotations

import os
import time
from dataclasses import dataclass, field

import numpy as np

from ..planning import catalog
from ..planning.costdb import ProfileDb, load_profile, synth_profile
from ..planning.faults import InfeasibleBudget, SpecError
from ..planning.graph import ModelSpec, ShardKind
from ..planning.hardware import MachineSpec
from ..planning.placement import TIERS, TierTable, TierEntry, reachable_tiers
from ..planning.pipeline_model import outstanding_tokens, schedule_iteration
from . import lib as L
from .executor import GEMV_MAX_T, Executor, PassSpec
from .model import HostWeights, arch_for


def _meminfo() -> dict:
    out = {}
    try:
        with open("/proc/meminfo") as fh:
            for line in fh:
                k, v = line.split(":", 1)
                out[k] = int(v.split()[0]) * 1024
    except (OSError, ValueError):
        pass
    return out


@dataclass
class GenerateResult:
    tokens: list                 # per request: np.int32 array of generated ids
    ttft_s: float
    tps: float
    e2el_s: float
    decode_tokens: int
    decode_time_s: float
    passes: list = field(default_factory=list)   # (tier, T, seconds, bytes streamed)
    migration_bytes: int = 0
    # tier switches: (from tier, to tier, live KV pages per layer, bytes the executor moved,
    # (h2d, d2h) bytes the migration model predicts)
    switches: list = field(default_factory=list)
    # per request: one character per computed position (prompt + gen - 1) naming the
    # numerics of the pass that computed it — "G" GEMM pass (bf16 activations), "P"
    # GEMV pass with the tcgen05 prefill attention, "D" decode-only GEMV pass. The
    # oracle applies the same rounding points (oracle/model_ref.py `modes`).
    row_modes: list = field(default_factory=list)


@dataclass
class _Session:
    """Loop state of one request batch (the counters of `simulate_inference`)."""
    prompts: list
    prompt_left: list
    gen_left: list
    fed: list                          # prompt tokens fed so far, per request
    out: list                          # tokens read back so far, per request
    pending_host: list = field(default_factory=list)   # sampling passes not read yet
    last_sampled: list | None = None
    last_rows: int = 1
    passes: list = field(default_factory=list)
    switches: list = field(default_factory=list)
    migration: int = 0
    ttft: float | None = None
    t_start: float = field(default_factory=time.perf_counter)
    modes: list = field(default_factory=list)        # per request: pass numerics per position


class Engine:
    """Plan + weights + executor for one model under one VRAM budget."""

    def __init__(self, model, budget_bytes: float, context_len: int, batch: int = 1,
                 machine="b200", profile: str | None = None, seed: int = 0,
                 max_tokens: int | None = None, chunk_bytes: int = 64 << 20,
                 checkpoint: str | None = None, shared_weights: str | None = None,
                 migration_aware: bool = False, striper=None, kv_page_seed: int | None = None,
                 host_format: str | None = None):
        """`model`: preset name or ModelSpec (random-init weights), or None with
        `checkpoint` = a directory holding config.json + safetensors, or a .gguf file
        (real weights, runtime/checkpoint.py, runtime/gguf.py). `shared_weights`: a /dev/shm segment name shared by
        the replicas of one node (one host copy of the weights per node)."""
        ckpt = None
        if checkpoint is not None:
            from .checkpoint import open_checkpoint, spec_from_hf_config
            ckpt = open_checkpoint(checkpoint)
            if model is None:
                model, ck_arch = spec_from_hf_config(ckpt.config, seed=seed)
        self.spec: ModelSpec = catalog.builtin_model(model) if isinstance(model, str) else model
        self.machine: MachineSpec = (catalog.builtin_machine(machine) if isinstance(machine, str)
                                     else machine)
        self.db: ProfileDb = load_profile(profile) if profile else synth_profile(self.machine)
        if striper is not None:   # N links feed this GPU: plan with the striped link model
            self.machine = catalog.striped_machine(self.machine, striper.n_helpers + 1)
        self.budget = float(budget_bytes)
        self.context_len = int(context_len)
        self.batch = int(batch)
        self.arch = arch_for(self.spec, seed)
        if ckpt is not None and ckpt.config:
            self.arch = spec_from_hf_config(ckpt.config, seed=seed)[1]
        # per-tier plans; tiers the budget cannot plan are unreachable (time = inf)
        self.plans = reachable_tiers(self.spec, self.machine, self.db, self.budget,
                                     self.context_len, self.batch)
        if not self.plans:
            raise InfeasibleBudget(self.budget, self.budget, "every token tier")
        self.table = None
        if set(self.plans) == set(TIERS):
            self.table = TierTable(self.spec.name, self.machine.name, self.budget,
                                   self.context_len,
                                   {t: TierEntry(t, p) for t, p in self.plans.items()})
        if host_format is None:
            host_format = self._auto_host_format(ckpt, shared_weights, striper)
        self.host_format = host_format
        self.weights = HostWeights(self.spec, self.arch, shared=shared_weights, host_format=host_format)
        t0 = time.perf_counter()
        if ckpt is not None:
            if self.weights.shared is None or self.weights.shared.creator:
                self.weights.load(ckpt)
                if self.weights.shared is not None:
                    self.weights.shared.mark_ready()
            else:
                self.weights.shared.wait_ready()
        else:
            self.weights.generate()
        self.load_seconds = time.perf_counter() - t0
        self.max_tokens = max_tokens
        self.chunk_bytes = chunk_bytes
        self.executor: Executor | None = None
        from .migration import MigrationModel
        self.migration = MigrationModel(self.spec, self.weights.layout, self.plans, self.context_len,
                                        self.batch)
        self.migration_aware = migration_aware
        self.striper = striper        # runtime.striping.StripeLeader: helper GPUs pull stripes
        self._sess: _Session | None = None
        # KV pages in seeded random order instead of lowest-first (tests: every kernel and
        # copy must follow the block table)
        self.kv_page_seed = kv_page_seed

    # -- tier selection over reachable tiers (pick_tier, planner.py:451-460) --
    def pick_tier(self, n_new: int) -> int:
        if n_new < 1:
            raise SpecError(f"batch_new_tokens must be >= 1, got {n_new}")
        best, best_cost = None, None
        for tier in TIERS:
            plan = self.plans.get(tier)
            if plan is None:
                continue
            cost = -(-n_new // tier) * plan.estimated_time
            if best_cost is None or cost < best_cost:
                best, best_cost = tier, cost
        return best

    def _auto_host_format(self, ckpt, shared_weights, striper) -> str:
        """'coded' (no bf16 host blob, runtime/model.py) when the bf16 blob and its coded
        copy do not fit host memory together but the coded copy alone does (Llama-3.3-70B
        on a 196 GB box: 141 + 106 GB), for a dense random-init model with a private host
        copy; else 'bf16'. PS_HOST_FORMAT overrides."""
        env = os.environ.get("PS_HOST_FORMAT")
        if env:
            return env
        if (self.spec.moe is not None or ckpt is not None or shared_weights is not None or striper is not None
                or os.environ.get("PS_CODED", "1") != "1"):
            return "bf16"
        from .model import WeightLayout
        lay = WeightLayout(self.spec, self.arch)
        avail = _meminfo().get("MemAvailable", 0)
        coded = lay.total_bytes * 3 // 4 + lay.embed_bytes
        if avail and coded > 0.5 * avail and coded < 0.75 * avail:
            return "coded"
        return "bf16"

    def _needs_coded12(self) -> bool:
        """The 12-bit coded copy serves what hx does not: CPU-placed (zero-copy) shards, and
        routed experts when the hx copy has none. Built when some plan places a shard on
        the CPU backend, for MoE models without hx experts, or when hx is off (PS_HX=0)."""
        from ..planning.vocab import Backend
        hx = getattr(self.weights, "hx", None)
        if os.environ.get("PS_HX", "1") == "0" or hx is None:
            return True
        if self.spec.moe is not None and (not hx.experts or os.environ.get("PS_HX_EXPERTS", "1") == "0"):
            return True
        return any(p.exec_backend is Backend.CPU for plan in self.plans.values() for p in plan.placements)

    def _build_hx(self) -> None:
        """hx copies (runtime/hxcodec.py, ~0.65 x the dense bytes, encoded on the GPU) of
        the dense shards: decode passes and prefill passes stream them, resident shards
        are held in that form. Node-shared with node-shared weights; skipped (bf16 /
        12-bit streaming) when host memory is short."""
        from .hxcodec import HxShards
        kinds = (ShardKind.ATTENTION, ShardKind.FFN, ShardKind.OUTPUT_HEAD, ShardKind.MOE_EXPERT_GROUP)
        dense = sum(b.nbytes for b in self.weights.layout.blobs.values() if b.kind in kinds)
        need = dense * 2 // 3
        shared = None
        meminfo = _meminfo()
        if self.weights.shared is not None:
            shared = os.path.basename(self.weights.shared.path) + "_hx"
        elif meminfo.get("MemAvailable", 0) and need > 0.5 * meminfo["MemAvailable"]:
            self.hx_skipped = "host memory: hx copy exceeds half of MemAvailable"
            return
        t0 = time.perf_counter()
        try:
            self.weights.hx = HxShards(self.weights, kinds, shared=shared)
        except Exception as exc:   # e.g. pinned host memory exhausted
            import warnings
            warnings.warn(f"hx-coded weights unavailable ({exc}); streaming without them")
            self.weights.hx = None
            self.hx_skipped = repr(exc)[:200]
            return
        self.hx_seconds = time.perf_counter() - t0

    def _build_coded(self) -> None:
        """Exponent-coded copies of the dense shards (runtime/wcomp.py) that decode
        passes stream instead of bf16 (25 % fewer link bytes, bit-identical results),
        when host memory holds them: about 0.75 x the dense weight bytes, pinned. With
        node-shared weights the coded copy is node-shared too (one replica encodes, the
        others map it), and the go / no-go rule uses only node totals, so every replica
        of a job decides the same. Anything else keeps bf16 streaming."""
        from .wcomp import CodedShards
        kinds = (ShardKind.ATTENTION, ShardKind.FFN, ShardKind.OUTPUT_HEAD, ShardKind.MOE_EXPERT_GROUP)
        dense = sum(b.nbytes for b in self.weights.layout.blobs.values() if b.kind in kinds)
        need = dense * 3 // 4
        shared = None
        meminfo = _meminfo()
        if self.weights.shared is not None:
            shared = os.path.basename(self.weights.shared.path) + "_coded"
            host_blob = self.weights.shared.nbytes
            if meminfo.get("MemTotal", 0) and need + host_blob > 0.8 * meminfo["MemTotal"]:
                self.coded_skipped = "node memory: bf16 + coded copies exceed 80 % of MemTotal"
                return
        elif meminfo.get("MemAvailable", 0) and need > 0.5 * meminfo["MemAvailable"]:
            self.coded_skipped = "host memory: coded copy exceeds half of MemAvailable"
            return
        t0 = time.perf_counter()
        try:
            self.weights.coded = CodedShards(self.weights, kinds, shared=shared)
        except Exception as exc:   # e.g. pinned host memory exhausted: stream bf16
            import warnings
            warnings.warn(f"exponent-coded weights unavailable ({exc}); streaming bf16")
            self.weights.coded = None
            self.coded_skipped = repr(exc)[:200]
            return
        self.coded_seconds = time.perf_counter() - t0
        self.coded_shared = shared is not None

    def _ensure_executor(self, max_tokens: int) -> Executor:
        if self.executor is None:
            tiers_used = self.plans
            if (os.environ.get("PS_CODED", "1") == "1" and os.environ.get("PS_HX", "1") != "0"
                    and getattr(self.weights, "hx", None) is None and self.weights.host_format == "bf16"):
                self._build_hx()
            if (os.environ.get("PS_CODED", "1") == "1" and getattr(self.weights, "coded", None) is None
                    and self.weights.host_format == "bf16" and self._needs_coded12()):
                self._build_coded()
            self.executor = Executor(self.weights, self.arch, tiers_used, self.budget,
                                     self.batch, self.context_len,
                                     self.max_tokens or max_tokens, chunk_bytes=self.chunk_bytes,
                                     kv_page_seed=self.kv_page_seed)
            self.migration.pins_fn = self.executor.pins_for   # include the spare pins
            self.migration.phys_fn = self.executor.phys_bytes  # coded-resident shards
            if self.striper is not None:
                if self.weights.shared is None:
                    raise SpecError("striped streaming needs node-shared weights (shared_weights=...)")
                self.striper.attach(self.executor.arena.base, self.weights.base,
                                    self.weights.shared.nbytes)
                self.executor.striper = self.striper
                if self.executor.ring is not None:
                    self.executor.ring.striper = self.striper
        elif max_tokens > self.executor.Tmax:
            raise SpecError(f"pass of {max_tokens} tokens exceeds the executor's {self.executor.Tmax}")
        return self.executor

    def attach_striper(self, prompt_lens: list, gen_len: int) -> None:
        """Create the executor now and export its arena to the stripe helpers (they
        must map it before the first striped piece); then wait for them."""
        self._ensure_executor(self.max_pass_tokens(prompt_lens, gen_len))
        self.striper.wait_helpers()

    def max_pass_tokens(self, prompt_lens: list, gen_len: int) -> int:
        """Largest T any pass of generate() will run (dry run of the loop)."""
        pl, gl = list(prompt_lens), [gen_len] * len(prompt_lens)
        biggest = 1
        while any(p > 0 for p in pl) or any(g > 0 for g in gl):
            tier = self.pick_tier(outstanding_tokens(pl, gl))
            step = schedule_iteration(tier, pl, gl)
            biggest = max(biggest, step.context_consumed + step.decoded)
        return biggest

    def prepare(self, prompt_lens: list, gen_len: int) -> int:
        """Create the executor and make the decode tier resident, as a serving
        engine sits between requests; returns the bytes moved. TTFT measured
        after this includes the switch into the prefill tier and back."""
        ex = self._ensure_executor(self.max_pass_tokens(prompt_lens, gen_len))
        return ex.set_tier(self.pick_tier(len(prompt_lens)))

    # ------------------------------------------------- one iteration at a time
    def submit(self, prompts: list, gen_len: int) -> None:
        """Start a request batch: `prompts` (one int array per request slot) each
        to be followed by `gen_len` greedy tokens. No GPU work; the batch then
        advances one reference iteration per `prefill()` / `decode()` call
        (`pkg/src/shardplan/simulator.py:273-297`), or all at once in `generate()`."""
        if not prompts:
            raise SpecError("generate needs at least one request")
        if len(prompts) > self.batch:
            raise SpecError(f"{len(prompts)} requests exceed the planned batch of {self.batch}")
        if gen_len < 1:
            raise SpecError(f"gen_len must be >= 1, got {gen_len}")
        prompts = [np.asarray(p, np.int32) for p in prompts]
        if min(len(p) for p in prompts) < 1:
            raise SpecError("every prompt needs at least one token")
        if max(len(p) for p in prompts) + gen_len > self.context_len:
            raise SpecError("prompt + gen exceeds the planned context length")
        self._ensure_executor(self.max_pass_tokens([len(p) for p in prompts], gen_len))
        self.executor.reset_requests()          # a new batch: free every KV page
        n = len(prompts)
        self._sess = _Session(prompts, [len(p) for p in prompts], [gen_len] * n, [0] * n,
                              [[] for _ in range(n)], modes=[""] * n)

    @property
    def outstanding(self) -> int:
        """New tokens the next iteration would be planned for (0: batch finished)."""
        s = self._sess
        return 0 if s is None else outstanding_tokens(s.prompt_left, s.gen_left)

    def prefill(self, prompts: list | None = None, gen_len: int | None = None) -> dict:
        """One iteration that consumes prompt tokens (a chunk of every unfinished
        prompt that fits the picked tier, plus one decode token of each request
        already past its prompt — the reference's mixed iteration). With
        `prompts`, starts a new batch first (`gen_len` defaults to 1). Returns
        {request slot: token id} of the requests whose final prompt chunk ran."""
        if prompts is not None:
            self.submit(prompts, 1 if gen_len is None else gen_len)
        s = self._need_session()
        if not any(p > 0 for p in s.prompt_left):
            raise SpecError("prefill(): no prompt tokens outstanding (call decode())")
        return self._finish_step(self._iterate())

    def decode(self) -> dict:
        """One decode-only iteration: one new token for every request that still
        has tokens to generate. Returns {request slot: token id}."""
        s = self._need_session()
        if any(p > 0 for p in s.prompt_left):
            raise SpecError("decode(): prompt tokens outstanding (call prefill())")
        if not any(g > 0 for g in s.gen_left):
            raise SpecError("decode(): every request has generated its tokens")
        return self._finish_step(self._iterate())

    def logits(self) -> np.ndarray:
        """fp32 logits [rows, V] of the last iteration's emitting requests, in slot order."""
        return self._need_executor().logits_host(self._sess.last_rows if self._sess else 1)

    def last_sampled_slots(self) -> list:
        """Request slots of the rows `logits()` returns (the last iteration's emitters)."""
        s = self._need_session()
        return list(s.last_sampled or [])

    def row_modes(self) -> list:
        """Per request: the numerics of the pass that computed each position so far
        (see GenerateResult.row_modes)."""
        return list(self._need_session().modes)

    def tokens(self) -> list:
        """Tokens generated so far, per request slot."""
        s = self._need_session()
        self._drain(self.executor, s.pending_host, s.out)
        return [np.array(o, np.int32) for o in s.out]

    def _need_session(self) -> "_Session":
        if getattr(self, "_sess", None) is None:
            raise SpecError("no request batch: call submit() or prefill(prompts)")
        return self._sess

    def _need_executor(self) -> Executor:
        if self.executor is None:
            raise SpecError("no pass has run yet")
        return self.executor

    def _finish_step(self, emitted: list) -> dict:
        s = self._sess
        self._drain(self.executor, s.pending_host, s.out)
        return {slot: int(s.out[slot][-1]) for slot in emitted}

    def _iterate(self, timing: bool = False, on_pass=None) -> list:
        """The loop body of `simulate_inference` (`simulator.py:273-297`) as one GPU
        pass: pick the tier for the outstanding new tokens (switching residency if it
        changes), feed prompt chunks / one decode token per request in request order,
        run the pass. Token ids are read back lazily; returns the emitting slots."""
        s, ex = self._sess, self.executor
        n = len(s.prompts)
        n_out = outstanding_tokens(s.prompt_left, s.gen_left)
        pages = ex.kv_live_pages()            # live KV pages per layer (what a switch moves)
        if self.migration_aware:
            tier = self.migration.pick_tier(n_out, ex.tier, pages, self.machine)
        else:
            tier = self.pick_tier(n_out)
        if tier != ex.tier:
            prev = ex.tier
            moved = ex.set_tier(tier)
            s.migration += moved
            s.switches.append((prev, tier, pages, moved, self.migration.bytes(prev, tier, pages)))
        step = schedule_iteration(tier, s.prompt_left, s.gen_left)
        slots, n_new, p0, ids, sample = [], [], [], [], []
        decode_ids_from_device = True
        for i in range(n):
            if step.prompt_take[i]:
                k = step.prompt_take[i]
                slots.append(i); n_new.append(k); p0.append(s.fed[i])
                ids.append(s.prompts[i][s.fed[i]:s.fed[i] + k])
                s.fed[i] += k
                decode_ids_from_device = False
            elif step.decode[i]:
                slots.append(i); n_new.append(1)
                p0.append(len(s.prompts[i]) + len(s.out[i]) - 1 + self._pending_count(s.pending_host, i))
                ids.append(None)
            if step.emits[i]:
                sample.append(len(slots) - 1)
        if decode_ids_from_device and s.last_sampled == slots:
            ids_arr = None
        else:
            self._drain(ex, s.pending_host, s.out)
            ids_arr = np.concatenate([a if a is not None else
                                      np.array([s.out[slots[j]][-1]], np.int32)
                                      for j, a in enumerate(ids)]).astype(np.int32)
            for j, a in enumerate(ids):      # decode positions are exact once drained
                if a is None:
                    p0[j] = len(s.prompts[slots[j]]) + len(s.out[slots[j]]) - 1
        T = sum(n_new)
        mode = "G" if T > GEMV_MAX_T else ("D" if all(k == 1 for k in n_new) else "P")
        for slot, k in zip(slots, n_new):
            s.modes[slot] += mode * k
        ev0 = L.event_create(True) if timing else 0
        if timing:
            L.call("ps_event_record", ev0, ex.cs)
        if on_pass is not None:
            on_pass(len(s.passes), tier, ex)       # e.g. attach / detach a tracer
        stats = ex.run_pass(PassSpec(slots, n_new, p0, ids_arr, sample))
        emitted = [slots[j] for j in sample]
        if sample:
            s.pending_host.append(emitted)
            s.last_sampled = emitted
            s.last_rows = len(sample)
        ev1 = 0
        if timing:
            ev1 = L.event_create(True)
            L.call("ps_event_record", ev1, ex.cs)
        s.passes.append([tier, stats.T, ev0, ev1, stats,   # bytes read after the final synchronize
                         step.context_consumed == 0 and step.decoded > 0, stats.zero_copy_bytes])
        if step.first_prompt_done and s.ttft is None:
            self._drain(ex, s.pending_host, s.out)   # first token is on the host
            s.ttft = time.perf_counter() - s.t_start
        ex.check_errors()
        return emitted

    # ------------------------------------------------------------------ generate
    def generate(self, prompts: list, gen_len: int, timing: bool = True,
                 on_pass=None) -> GenerateResult:
        """Greedy generation for a batch of prompts: `submit` then the reference
        loop (`simulator.py:273-297`) of `prefill()` / `decode()` iterations until
        every request has its `gen_len` tokens, with tokens read back lazily."""
        self.submit(prompts, gen_len)
        s, ex = self._sess, self.executor
        s.t_start = time.perf_counter()
        while outstanding_tokens(s.prompt_left, s.gen_left):
            self._iterate(timing, on_pass)
        self._drain(ex, s.pending_host, s.out)
        ex.synchronize()
        ex.check_errors()
        total = time.perf_counter() - s.t_start
        decode_time, decode_tokens = 0.0, 0
        pass_rows = []
        for tier, T, e0, e1, st, is_decode, zc in s.passes:
            nbytes = st.bytes_streamed    # settled: speculative fetches count what crossed
            secs = L.event_elapsed_ms(e0, e1) / 1e3 if timing else float("nan")
            # (tier, tokens, seconds, bytes via the copy engine, bytes read zero-copy)
            pass_rows.append((tier, T, secs, nbytes, zc))
            if is_decode:
                decode_tokens += T
                decode_time += secs
            if timing:
                L.call("ps_event_destroy", e0)
                L.call("ps_event_destroy", e1)
        ttft = total if s.ttft is None else s.ttft
        tps = decode_tokens / decode_time if decode_time > 0 else float("inf")
        return GenerateResult([np.array(o, np.int32) for o in s.out], ttft, tps,
                              ttft + 100.0 / tps if tps else float("inf"),
                              decode_tokens, decode_time, pass_rows, s.migration, s.switches,
                              list(s.modes))

    @staticmethod
    def _pending_count(pending_host, slot) -> int:
        return sum(1 for slots in pending_host if slot in slots)

    @staticmethod
    def _drain(ex, pending_host, out) -> None:
        if not pending_host:
            return
        for slots, toks in ex.collect_tokens():
            for s, t in zip(slots, toks):
                out[s].append(int(t))
        pending_host.clear()

    def close(self) -> None:
        if self.executor is not None:
            self.executor.close()
            self.executor = None
        coded = getattr(self.weights, "coded", None)
        if coded is not None:
            coded.close()
            self.weights.coded = None
        hx = getattr(self.weights, "hx", None)
        if hx is not None:
            hx.close()
            self.weights.hx = None
        self.weights.close()
