"""Sweep GEMV work decompositions on the shapes a decode pass launches.

Times each launch with CUDA events on its stream, L2 flushed between launches.
Prints achieved GB/s (algorithmic bytes: weights + x + y) per config."""
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L

SHAPES = [(6144, 4096, "wqkv piece"), (4096, 4096, "wo piece"), (8192, 4096, "wgu/lm piece 64MB"),
          (2340, 14336, "wdown piece"), (28672, 4096, "wgu full 235MB"), (4096, 14336, "wdown full")]
CFGS = [(0, 0, 0), (0, 0, 296), (2, 0, 0), (2, 8, 0), (4, 8, 0)]


def run(N, K, rows, ks, grid, t=1, epi=0, reps=10):
    W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_()
    x = torch.randn(t, K, device="cuda")
    y = torch.zeros(t, N, device="cuda")
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB > L2
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(reps + 2):
        flush.sum()
        e0.record()
        L.call("ps_gemv_bf16_cfg", x.data_ptr(), K, t, W.data_ptr(), N, K, K, y.data_ptr(), N, epi, s,
               rows, ks, grid)
        e1.record()
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(e0.elapsed_time(e1) / 1e3)
    ref = x @ W.float().T
    err = float((y - ref).abs().max() / ref.abs().max())
    nbytes = N * K * 2 + t * K * 4 + t * N * 4
    avg = sum(ts) / len(ts)
    return nbytes / avg / 1e9, avg * 1e6, err


out = []
for N, K, name in SHAPES:
    for rows, ks, grid in CFGS:
        gbs, us, err = run(N, K, rows, ks, grid)
        out.append({"shape": name, "N": N, "K": K, "rows": rows, "ksplit": ks, "grid": grid,
                    "GBps": round(gbs, 1), "us": round(us, 2), "err": err})
        print(json.dumps(out[-1]), flush=True)
for t in (2, 4, 8, 32):
    for rows in (0, 2):
        gbs, us, err = run(28672, 4096, rows, 0, 0, t=t)
        print(json.dumps({"shape": f"wgu full t={t}", "rows": rows, "GBps": round(gbs, 1), "us": round(us, 2),
                          "err": err}))
