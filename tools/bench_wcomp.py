"""Exponent-coded weights (runtime/wcomp.py): coded GEMV `ps_gemv_bf16c` vs bf16 GEMV
`ps_gemv_bf16` (t <= 8; ps_gemv_tc, the one-pass tcgen05 kernel, for t > 8) on L8 shapes (random-init weights of the oracle initialiser, the head
with its heavy-tailed rows), t in {1, 2, 4, 8}, plus host -> device time of a 64 MB ring
piece as bf16 vs coded. Weights rotate over copies totalling > L2 (126 MB), so every
launch reads HBM. Prints one JSON line per case; `frac` = coded bytes / time / HBM peak."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import model_ref as M  # noqa: E402
from paper_2604_26334_b200.runtime import lib as L, wcomp  # noqa: E402

PEAK = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6547.5
s = torch.cuda.current_stream().cuda_stream
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def timed(fns, reps=30):
    ts = []
    for i in range(reps + 3):
        fn = fns[i % len(fns)]
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def case(name, tensor, N, K, ts=(1, 2, 4, 8)):
    bits = M.bf16_bits(0, tensor, N, K)
    coded, tb = wcomp.encode(bits)
    copies = max(2, -(-(300 << 20) // coded.nbytes))
    dc = [torch.from_numpy(coded).cuda() for _ in range(copies)]
    db = [torch.from_numpy(bits.view(np.int16)).cuda() for _ in range(copies)]
    n_esc = int((coded[:, K * 3 // 2:].copy().view(np.uint32)[:, 0] >> 8).sum())
    for t in ts:
        x = torch.randn(t, K, device="cuda")
        y = torch.zeros(t, N, device="cuda")
        if t <= 8:
            tc = timed([lambda w=w: L.call("ps_gemv_bf16c", x.data_ptr(), K, t, w.data_ptr(), N, K, coded.shape[1],
                                           y.data_ptr(), N, 0, s) for w in dc])
            tbf = timed([lambda w=w: L.call("ps_gemv_bf16", x.data_ptr(), K, t, w.data_ptr(), N, K, K, y.data_ptr(),
                                            N, 0, s) for w in db])
        else:   # one-pass tensor-core GEMV (ps_gemv_tc), coded and bf16
            ws_n = ctypes.c_longlong()
            L.call("ps_gemv_tc_workspace", N, K, ctypes.byref(ws_n))
            ws = torch.empty(ws_n.value, dtype=torch.uint8, device="cuda")
            tc = timed([lambda w=w: L.call("ps_gemv_tc", x.data_ptr(), K, t, w.data_ptr(), N, K, coded.shape[1], 1,
                                           y.data_ptr(), N, 0, ws.data_ptr(), ws.numel(), s) for w in dc])
            tbf = timed([lambda w=w: L.call("ps_gemv_tc", x.data_ptr(), K, t, w.data_ptr(), N, K, K, 0,
                                            y.data_ptr(), N, 0, ws.data_ptr(), ws.numel(), s) for w in db])
        gb = coded.nbytes / tc / 1e3
        print(json.dumps({"case": name, "N": N, "K": K, "t": t, "trailer": tb, "escapes": n_esc,
                          "coded_bytes": coded.nbytes, "bf16_bytes": bits.nbytes, "coded_us": round(tc, 2),
                          "bf16_us": round(tbf, 2), "coded_gbs": round(gb, 1), "frac": round(gb / PEAK, 3),
                          "bf16_gbs": round(bits.nbytes / tbf / 1e3, 1)}), flush=True)
    return bits, coded


bits, coded = case("ffn piece 64MB", "L0.w_gate", 8192, 4096, ts=(1, 2, 4, 8, 32))
case("wgu 235MB", "L0.w_up", 28672, 4096, ts=(1, 8, 16, 32))
case("wdown", "L0.w_down", 4096, 14336, ts=(1, 32))
case("lm_head (heavy rows)", "lm_head", 32768, 4096, ts=(1,))
nb, nc = bits.nbytes, coded.nbytes
hb, hc = L.host_alloc(nb, mapped=False), L.host_alloc(nc, mapped=False)
ctypes.memmove(hb, bits.ctypes.data, nb)
ctypes.memmove(hc, coded.ctypes.data, nc)
db, dcc = torch.empty(nb, dtype=torch.uint8, device="cuda"), torch.empty(nc, dtype=torch.uint8, device="cuda")
h2d_b = timed([lambda: L.memcpy_async(db.data_ptr(), hb, nb, s)], 10)
h2d_c = timed([lambda: L.memcpy_async(dcc.data_ptr(), hc, nc, s)], 10)
print(json.dumps({"case": "h2d 64MB piece", "bf16_us": round(h2d_b, 1), "coded_us": round(h2d_c, 1),
                  "link_time_ratio": round(h2d_c / h2d_b, 4)}))
