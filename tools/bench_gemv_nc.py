"""A/B of the bulk-copy GEMV (bf16 rows: ps_gemv_bf16, exponent-coded rows: ps_gemv_bf16c)
across builds of libpshard (PSHARD_LIB=...): decode shapes at t = 1, 2, 4, 8, L2 flushed
between launches, CUDA events on the launching stream. One JSON line per (shape, t, kind):
achieved GB/s over the algorithmic bytes (weights as stored + x + y)."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.runtime import lib as L, wcomp  # noqa: E402

SHAPES = [(28672, 4096, "wgu 235MB"), (4096, 14336, "wdown"), (8192, 4096, "64MB piece"), (6144, 4096, "wqkv")]
tag = sys.argv[1] if len(sys.argv) > 1 else os.environ.get("PSHARD_LIB", "default")
s = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=12):
    ts = []
    for i in range(reps + 2):
        flush.sum()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    return sorted(ts)[len(ts) // 2]


for N, K, name in SHAPES:
    W = ((torch.rand(N, K, device="cuda", generator=g) * 2 - 1) * math.sqrt(3 / K)).to(torch.bfloat16)
    coded, _ = wcomp.encode(W.view(torch.int16).cpu().numpy().view(np.uint16))
    Wc = torch.from_numpy(coded).cuda()
    rb = coded.shape[1]
    for t in (1, 2, 4, 8):
        x = torch.randn(t, K, device="cuda", generator=g)
        ya, yb = torch.zeros(t, N, device="cuda"), torch.zeros(t, N, device="cuda")
        ta = timed(lambda: L.call("ps_gemv_bf16", x.data_ptr(), K, t, W.data_ptr(), N, K, K, ya.data_ptr(), N, 0, s))
        tb = timed(lambda: L.call("ps_gemv_bf16c", x.data_ptr(), K, t, Wc.data_ptr(), N, K, rb, yb.data_ptr(), N, 0,
                                  s))
        same = bool(torch.equal(ya, yb))
        io = t * K * 4 + t * N * 4
        for kind, sec, nb in (("bf16", ta, N * K * 2 + io), ("coded", tb, N * rb + io)):
            print(json.dumps({"lib": tag, "shape": name, "N": N, "K": K, "t": t, "kind": kind,
                              "us": round(sec * 1e6, 2), "GBps": round(nb / sec / 1e9, 1),
                              "bit_identical": same}), flush=True)
