"""Zero-copy GEMV configurations on a host-mapped matrix (the tiny config's CPU-placed
head, 32000 x 512 bf16 = 32.8 MB, and an L8-shaped 4096 x 4096 piece): GB/s per
(rows per warp, k-split, grid cap); rows = -1 is the bulk-copy kernel reading host memory.

    python tools/zc_gemv_sweep.py"""
import ctypes
import json
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L  # noqa: E402

CFGS = [(0, 0, 0), (-1, 0, 0), (2, 1, 0), (4, 1, 0), (2, 2, 0), (4, 2, 0), (2, 1, 296), (4, 1, 296),
        (2, 1, 592), (4, 1, 592), (2, 4, 0)]
for N, K in ((32000, 512), (4096, 4096)):
    nbytes = N * K * 2
    host = L.host_alloc(nbytes, mapped=True)
    src = torch.randn(N, K).to(torch.bfloat16)
    ctypes.memmove(host, src.data_ptr(), nbytes)
    x = torch.randn(1, K, device="cuda")
    y = torch.zeros(1, N, device="cuda")
    ref = (x.cpu() @ src.float().T)
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for rows, ks, grid in CFGS:
        ts = []
        try:
            for i in range(7):
                e0.record()
                L.call("ps_gemv_bf16_cfg", x.data_ptr(), K, 1, host, N, K, K, y.data_ptr(), N, 0, s, rows, ks, grid)
                e1.record()
                torch.cuda.synchronize()
                if i >= 2:
                    ts.append(e0.elapsed_time(e1) / 1e3)
        except Exception as exc:   # unsupported combination
            print(json.dumps({"N": N, "K": K, "rows": rows, "ksplit": ks, "grid": grid, "error": str(exc)[:80]}))
            continue
        err = float((y.cpu() - ref).abs().max() / ref.abs().max())
        t = min(ts)
        print(json.dumps({"N": N, "K": K, "rows": rows, "ksplit": ks, "grid": grid,
                          "GBps": round(nbytes / t / 1e9, 1), "us": round(t * 1e6, 1), "err": err}))
    L.host_free(host)
