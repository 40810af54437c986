"""Does the L2 keep host-mapped (zero-copy) data? Time a zero-copy GEMV over a
host matrix twice back to back (no flush between), and after a prefetch pass."""
import ctypes, json, sys
import torch
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L

N, K = 32000, 512
nbytes = N * K * 2
host = L.host_alloc(nbytes, mapped=True)
ctypes.memset(host, 0x3c, nbytes)
x = torch.randn(1, K, device="cuda"); y = torch.zeros(1, N, device="cuda")
flush = torch.ones(64 << 20, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def t(rows, note):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    L.call("ps_gemv_bf16_cfg", x.data_ptr(), K, 1, host, N, K, K, y.data_ptr(), N, 0, s, rows, 0, 0)
    e1.record(); torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3
    print(json.dumps({"note": note, "rows": rows, "us": round(us, 1), "GBps": round(nbytes / us / 1e3, 1)}), flush=True)
for rows in (2, -1):
    for rep in range(3):
        flush.sum(); torch.cuda.synchronize()
        t(rows, "cold (L2 flushed)")
        t(rows, "warm (same matrix again)")
L.host_free(host)
