"""Measured install phase: time the real sm_100a kernels on the benchmark grid
and write a `shardplan-profile v1` file the planner can load.

The reference's install phase is synthetic (`pkg/src/shardplan/profile_db.py:192-261`
derives every entry from the machine's roofline curves); the paper's is
measured — each kernel shape is launched 10 times asynchronously and the
average taken (`PAPER.md:227-228`). This module is that measured phase for
this build: every GPU grid point of the `f16` class (the class bf16 weights
snap to, `pkg/src/shardplan/kernels.py:50-54`) is timed on the kernel the
executor actually launches for it:

| op (grid dims)                     | kernel                                             |
|------------------------------------|----------------------------------------------------|
| MATMUL (m, k, n), m <= 32          | ps_gemv_bf16, fp32 activations                     |
| MATMUL (m, k, n), m > 32           | ps_gemm_bf16 (CTA-pair tcgen05), rows in <= 16384 slices |
| GQA / MHA (t, ctx, ...), t <= 32   | ps_attn_decode, t requests at length ctx           |
| GQA / MHA (t, ctx, ...), t > 32    | ps_attn_prefill_tc, ceil(t / ctx) requests, causal |
| MOE_ROUTE (t, d, E)                | router matmul + ps_moe_route_topk (k = 8)          |
| ELEMENT_WISE (n,)                  | ps_rmsnorm over n / 4096 rows                      |

Entry rates are the canonical workload (`canonical_workload`, the same FLOP /
byte accounting the planner prices requests with) divided by the measured
time, so an exact hit returns the measured time and a nearest-neighbour hit
prices a nearby shape on the measured roofline. CPU entries and the other
quant classes have no kernel here (there is no CPU backend; bf16 is the only
weight format) and keep their synthesized values; the header says
`generator measured` and a JSON sidecar records every measured point.

Weights and KV caches are cycled through enough copies that the working set
of the 10 timed launches exceeds L2 (126 MB), as in a decode pass where each
matrix is read once.

    python -m paper_2604_26334_b200.runtime.profiler --machine b200 --out b200.profile
"""

from __future__ import annotations

import argparse
import json
import math
import time
from dataclasses import dataclass

from ..planning import catalog
from ..planning.costdb import (Generator, KernelKey, ProfileDb, ProfileEntry, ProfileMeta,
                               grid_shapes, machine_stamp, save_profile, synth_profile)
from ..planning.hardware import MachineSpec
from ..planning.vocab import Backend, OpKind, QUANT_CLASSES, canonical_workload

MEASURED_QUANT = "f16"
LAUNCHES = 10           # timed asynchronous launches per grid point
WARMUP = 2
L2_BYTES = 126 << 20
MAX_GEMM_ROWS = 16384   # the largest token tier (planner TIERS) — larger m runs in slices


@dataclass
class Point:
    op: str
    dims: tuple
    kernel: str
    seconds: float
    flops: float
    bytes: float
    method: str = ""


def _copies(nbytes: int, cap: int = 64) -> int:
    """Buffers to cycle so LAUNCHES launches touch more than L2."""
    return max(1, min(cap, math.ceil(2 * L2_BYTES / max(1, nbytes))))


class KernelBench:
    """Builds the inputs of one grid point and times LAUNCHES launches of its
    kernel back to back on one stream (CUDA events around the batch)."""

    def __init__(self, graphs: bool = True):
        import torch

        from . import lib as L
        self.torch, self.L = torch, L
        if not torch.cuda.is_available():
            raise RuntimeError("the measured profiler needs a GPU")
        self.graphs = graphs
        self.method = None

    @property
    def stream(self) -> int:
        # the current stream at launch time: inside graph capture it is the capture stream
        return self.torch.cuda.current_stream().cuda_stream

    def _time(self, launch, n_variants: int) -> float:
        """Seconds per launch. The LAUNCHES launches are captured in a CUDA graph
        and replayed, so the host's per-call cost (ctypes) cannot starve the GPU
        between small kernels — as in a decode pass, where the host enqueues the
        whole pass ahead of the copy engine. Best of 3 replays."""
        torch, L = self.torch, self.L
        for i in range(WARMUP):
            launch(i % n_variants)
        torch.cuda.synchronize()
        best = None
        if self.graphs:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    for i in range(LAUNCHES):
                        launch(i % n_variants)
                g.replay()
                for _ in range(3):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    g.replay()
                    e1.record()
                    e1.synchronize()
                    t = e0.elapsed_time(e1) / 1e3 / LAUNCHES
                    best = t if best is None else min(best, t)
                self.method = "cuda-graph replay of 10 launches, best of 3"
                del g
                return best
            except RuntimeError:
                torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(LAUNCHES):
            launch(i % n_variants)
        e1.record()
        e1.synchronize()
        self.method = "10 asynchronous launches"
        return e0.elapsed_time(e1) / 1e3 / LAUNCHES

    # -- one method per op kind: returns (kernel name, seconds per launch) -------------
    def matmul(self, m: int, k: int, n: int):
        torch, L = self.torch, self.L
        nw = _copies(n * k * 2)
        Ws = [torch.empty(n, k, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02) for _ in range(nw)]
        if m <= 32:
            x = torch.randn(m, k, device="cuda")
            y = torch.empty(m, n, device="cuda")

            def launch(i):
                L.call("ps_gemv_bf16", x.data_ptr(), k, m, Ws[i].data_ptr(), n, k, k, y.data_ptr(), n,
                       L.PS_EPI_STORE, self.stream)
            return "ps_gemv_bf16", self._time(launch, nw)
        rows = min(m, MAX_GEMM_ROWS)
        slices = math.ceil(m / rows)
        A = torch.randn(rows, k, device="cuda").to(torch.bfloat16)
        C = torch.empty(rows, n, device="cuda")

        def launch(i):
            for j in range(slices):
                r = min(rows, m - j * rows)
                L.call("ps_gemm_bf16", A.data_ptr(), r, k, k, Ws[i].data_ptr(), n, k, C.data_ptr(), n,
                       L.PS_EPI_STORE, self.stream)
        return "ps_gemm_bf16" + (f" x{slices} row slices" if slices > 1 else ""), self._time(launch, nw)

    def attention(self, t: int, ctx: int, heads: int, kv: int, hd: int):
        torch, L = self.torch, self.L
        qrows = (heads + 2 * kv) * hd
        row_elems = 2 * kv * hd
        page = 64
        pps = -(-ctx // page)

        def table(n_req):   # request b owns pages [b * pps, (b + 1) * pps) of the pool
            return torch.arange(n_req * pps, dtype=torch.int32, device="cuda").view(n_req, pps)
        if t <= 32:
            B = t
            ncache = _copies(pps * page * B * row_elems * 2, cap=8)
            caches = [torch.empty(pps * page * B * row_elems, dtype=torch.bfloat16, device="cuda").normal_()
                      for _ in range(ncache)]
            bt = table(B)
            q = torch.randn(B, qrows, device="cuda")
            out = torch.empty(B, heads * hd, device="cuda")
            lens = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
            ws_floats = L.attn_decode_workspace(B, heads, hd, ctx)
            ws = torch.empty(max(1, ws_floats), device="cuda")

            def launch(i):
                L.call("ps_attn_decode", q.data_ptr(), qrows, B, heads, kv, hd, 0, caches[i].data_ptr(),
                       row_elems, bt.data_ptr(), pps, page, lens.data_ptr(), ctx, 1.0 / math.sqrt(hd),
                       out.data_ptr(), heads * hd, ws.data_ptr(), ws_floats, self.stream)
            return "ps_attn_decode", self._time(launch, ncache)
        nreq = math.ceil(t / ctx)
        new = [min(ctx, t - i * ctx) for i in range(nreq)]
        q_start = [0]
        for v in new:
            q_start.append(q_start[-1] + v)
        p0 = [ctx - v for v in new]
        cache = torch.empty(pps * page * nreq * row_elems, dtype=torch.bfloat16, device="cuda").normal_()
        bt = table(nreq)
        q = torch.randn(t, qrows, device="cuda")
        out = torch.empty(t, heads * hd, dtype=torch.bfloat16, device="cuda")
        i_qs = torch.tensor(q_start, dtype=torch.int32, device="cuda")
        i_p0 = torch.tensor(p0, dtype=torch.int32, device="cuda")

        def launch(i):
            L.call("ps_attn_prefill_tc", q.data_ptr(), qrows, nreq, i_qs.data_ptr(), i_p0.data_ptr(), 0,
                   max(new), heads, kv, hd, cache.data_ptr(), row_elems, bt.data_ptr(), pps, page, nreq * pps,
                   1.0 / math.sqrt(hd), out.data_ptr(), heads * hd, 1, self.stream)
        return "ps_attn_prefill_tc", self._time(launch, 1)

    def moe_route(self, t: int, d: int, E: int, top_k: int = 8):
        torch, L = self.torch, self.L
        nw = _copies(E * d * 2)
        Ws = [torch.empty(E, d, dtype=torch.bfloat16, device="cuda").normal_(0, 0.02) for _ in range(nw)]
        logits = torch.empty(t, E, device="cuda")
        ids = torch.empty(t, top_k, dtype=torch.int32, device="cuda")
        w = torch.empty(t, top_k, device="cuda")
        if t <= 32:
            x = torch.randn(t, d, device="cuda")
        else:
            x = torch.randn(t, d, device="cuda").to(torch.bfloat16)

        def launch(i):
            if t <= 32:
                L.call("ps_gemv_bf16", x.data_ptr(), d, t, Ws[i].data_ptr(), E, d, d, logits.data_ptr(), E,
                       L.PS_EPI_STORE, self.stream)
            else:
                L.call("ps_gemm_bf16", x.data_ptr(), t, d, d, Ws[i].data_ptr(), E, d, logits.data_ptr(), E,
                       L.PS_EPI_STORE, self.stream)
            L.call("ps_moe_route_topk", logits.data_ptr(), E, t, E, top_k, 1, ids.data_ptr(), w.data_ptr(), self.stream)
        return "router matmul + ps_moe_route_topk", self._time(launch, nw)

    def elementwise(self, n: int):
        torch, L = self.torch, self.L
        d = min(n, 4096)
        rows = max(1, n // d)
        nb = _copies(n * 4, cap=16)
        xs = [torch.randn(rows, d, device="cuda") for _ in range(nb)]
        wt = torch.ones(d, dtype=torch.bfloat16, device="cuda")
        out = torch.empty(rows, d, device="cuda")

        def launch(i):
            L.call("ps_rmsnorm", xs[i].data_ptr(), d, 0, rows, wt.data_ptr(), d, 1e-5, out.data_ptr(), d, 0, self.stream)
        return "ps_rmsnorm", self._time(launch, nb)

    def run(self, op: OpKind, dims: tuple):
        if op is OpKind.MATMUL:
            return self.matmul(*dims)
        if op is OpKind.GQA:
            return self.attention(*dims)
        if op is OpKind.MHA:
            t, ctx, h, hd = dims
            return self.attention(t, ctx, h, h, hd)
        if op is OpKind.MOE_ROUTE:
            return self.moe_route(*dims)
        if op is OpKind.ELEMENT_WISE:
            return self.elementwise(*dims)
        raise ValueError(f"no kernel for {op}")


def measure_points(shapes=None, bench=None, log=None) -> list[Point]:
    """Time the f16 GPU grid points (all of `grid_shapes()` unless `shapes`)."""
    bench = bench or KernelBench()
    bpe = QUANT_CLASSES[MEASURED_QUANT]
    out = []
    for op, dims in (shapes if shapes is not None else grid_shapes()):
        flops, byts = canonical_workload(op, dims, bpe)
        kernel, secs = bench.run(op, dims)
        if not secs > 0:
            raise RuntimeError(f"non-positive time for {op.value}{dims}")
        out.append(Point(op.value, tuple(dims), kernel, secs, flops, byts, getattr(bench, "method", "") or ""))
        if log:
            log(out[-1])
        try:
            bench.torch.cuda.empty_cache()
        except AttributeError:
            pass
    return out


def measured_profile(machine: MachineSpec, points: list[Point]) -> ProfileDb:
    """The synthetic profile of `machine` with every measured (GPU, f16) entry
    replaced by its measured rates."""
    measured = {(OpKind(p.op), p.dims): p for p in points}
    entries = []
    for e in synth_profile(machine).entries():
        k = e.key
        p = measured.get((k.op_kind, k.dims))
        if k.backend is Backend.GPU and k.quant == MEASURED_QUANT and p is not None:
            e = ProfileEntry(KernelKey(k.op_kind, k.quant, k.backend, 0, k.dims),
                             flops_per_sec=p.flops / p.seconds if p.flops > 0 else p.bytes / p.seconds,
                             bytes_per_sec=p.bytes / p.seconds)
        entries.append(e)
    meta = ProfileMeta(machine_id=machine.name, generation_timestamp=machine_stamp(machine),
                       generator=Generator.MEASURED)
    return ProfileDb(entries, meta)


def write_sidecar(path: str, machine: MachineSpec, points: list[Point]) -> None:
    doc = {"machine": machine.name, "launches_per_point": LAUNCHES, "warmup": WARMUP,
           "measured_quant": MEASURED_QUANT, "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "points": [{"op": p.op, "dims": list(p.dims), "kernel": p.kernel, "method": p.method,
                       "us": round(p.seconds * 1e6, 3),
                       "tflops": round(p.flops / p.seconds / 1e12, 3),
                       "gbps": round(p.bytes / p.seconds / 1e9, 2)} for p in points]}
    with open(path, "w") as fh:
        json.dump(doc, fh, indent=1)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--machine", default="b200")
    ap.add_argument("--out", required=True)
    ap.add_argument("--sidecar", help="JSON of the measured points (default: <out>.json)")
    ap.add_argument("--quick", action="store_true", help="every 3rd grid point only (smoke)")
    args = ap.parse_args(argv)
    machine = catalog.builtin_machine(args.machine)
    shapes = grid_shapes()
    if args.quick:
        shapes = shapes[::3]
    points = measure_points(shapes, log=lambda p: print(
        f"{p.op:12s} {str(p.dims):28s} {p.kernel:34s} {p.seconds * 1e6:10.2f} us "
        f"{p.flops / p.seconds / 1e12:8.2f} TF/s {p.bytes / p.seconds / 1e9:9.1f} GB/s", flush=True))
    db = measured_profile(machine, points)
    save_profile(db, args.out)
    write_sidecar(args.sidecar or args.out + ".json", machine, points)
    print(f"wrote {args.out}: {len(db)} entries, {len(points)} measured")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
