"""Exponent-coded weights on the link: host -> device time of a 64 MB L8-shaped ring
piece (8192 x 4096) as bf16 vs coded (12 bits/weight), plus the GEMV on each
(`ps_gemv_bf16` vs `ps_gemv_bf16c`), on the real random-init weights of L8's
w_gate (oracle initialiser). Prints JSON."""
import ctypes
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import model_ref as M  # noqa: E402
from paper_2604_26334_b200.runtime import lib as L, wcomp  # noqa: E402

N, K = 8192, 4096
bits = M.bf16_bits(0, "L0.w_gate", N, K)
coded, base, off, ent = wcomp.encode(bits)
nb, nc = bits.nbytes, coded.nbytes
hb = L.host_alloc(nb, mapped=False)
hc = L.host_alloc(nc, mapped=False)
ctypes.memmove(hb, bits.ctypes.data, nb)
ctypes.memmove(hc, coded.ctypes.data, nc)
db = torch.empty(nb, dtype=torch.uint8, device="cuda")
dc = torch.empty(nc, dtype=torch.uint8, device="cuda")
d_off, d_ent = torch.from_numpy(off).cuda(), torch.from_numpy(ent).cuda()
x = torch.randn(1, K, device="cuda")
y = torch.zeros(1, N, device="cuda")
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fn, reps=20):
    ts = []
    for i in range(reps + 3):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return min(ts)


out = {"shape": [N, K], "base": base, "escapes": int(len(ent)), "bf16_bytes": nb, "coded_bytes": int(nc + off.nbytes + ent.nbytes)}
out["h2d_bf16_us"] = timed(lambda: L.memcpy_async(db.data_ptr(), hb, nb, s))
out["h2d_coded_us"] = timed(lambda: L.memcpy_async(dc.data_ptr(), hc, nc, s))
out["gemv_bf16_us"] = timed(lambda: L.call("ps_gemv_bf16", x.data_ptr(), K, 1, db.data_ptr(), N, K, K, y.data_ptr(), N, 0, s))
out["gemv_coded_us"] = timed(lambda: L.call("ps_gemv_bf16c", x.data_ptr(), K, 1, dc.data_ptr(), N, K, base, d_off.data_ptr(),
                                            d_ent.data_ptr(), y.data_ptr(), N, 0, s))
out["link_time_ratio"] = round(out["h2d_coded_us"] / out["h2d_bf16_us"], 4)
print(json.dumps(out))
