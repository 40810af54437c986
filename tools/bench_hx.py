"""ps_hx_expand throughput (csrc/hx.cu): decode an hx-coded matrix to bf16 in VRAM, whole
and in expand-buffer-sized runs of 64-row blocks, L2 flushed between launches, CUDA
events on the launching stream. Prints one JSON line per case: coded GB/s read and
bf16 GB/s written."""
import json
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.runtime import hxcodec as hx, lib as L  # noqa: E402

s = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=10):
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


for N, K in [(28672, 4096), (4096, 14336), (6144, 4096)]:
    W = ((torch.rand(N, K, device="cuda", generator=g) * 2 - 1) * math.sqrt(3 / K)).to(torch.bfloat16)
    enc = hx.GpuHxEncoder()
    fill = lambda dst, r0, r1: L.memcpy_async(dst, W.data_ptr() + r0 * K * 2, (r1 - r0) * K * 2, s)  # noqa: E731
    m = enc.plan(fill, N, K)
    host = L.host_alloc(m.nbytes, mapped=False)
    enc.write(fill, m, host)
    blob = torch.empty(m.nbytes, dtype=torch.uint8, device="cuda")
    L.memcpy_async(blob.data_ptr(), host, m.nbytes, s)
    torch.cuda.synchronize()
    L.host_free(host)
    lut = torch.from_numpy(m.lut.view(np.int32)).cuda()
    out = torch.empty(N, K, dtype=torch.bfloat16, device="cuda")
    for run_rows in (N, 3584, 1024):
        run_rows = min(N, run_rows)
        offs = []
        for r0 in range(0, N, run_rows):
            ba, bb = r0 // 64, -(-min(N, r0 + run_rows) // 64)
            offs.append((r0, min(N, r0 + run_rows), int(m.block_off[ba]),
                         torch.from_numpy((m.block_off[ba:bb] - m.block_off[ba]).astype(np.int32)).cuda()))

        def run():
            for r0, r1, b0, rel in offs:
                L.call("ps_hx_expand", blob.data_ptr() + b0, rel.data_ptr(), r1 - r0, K, lut.data_ptr(),
                       out.data_ptr() + r0 * K * 2, K, s)
        sec = timed(run)
        ok = bool(torch.equal(out, W))
        print(json.dumps({"N": N, "K": K, "run_rows": run_rows, "launches": len(offs), "us": round(sec * 1e6, 1),
                          "coded_GBps": round(m.nbytes / sec / 1e9, 1), "bf16_out_GBps": round(N * K * 2 / sec / 1e9, 1),
                          "bits_per_weight": round(m.nbytes * 8 / (N * K), 3), "exact": ok}), flush=True)
