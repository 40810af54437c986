"""Zero-copy (host-mapped) read bandwidth of the GEMV kernel vs the copy engine."""
import ctypes, json, sys, time
import torch
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L

def run(N, K, rows=0, ks=0, grid=0, reps=5):
    nbytes = N * K * 2
    host = L.host_alloc(nbytes, mapped=True)
    ctypes.memset(host, 0x3c, nbytes)
    x = torch.randn(1, K, device="cuda"); y = torch.zeros(1, N, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 0
    for _ in range(reps):
        e0.record()
        L.call("ps_gemv_bf16_cfg", x.data_ptr(), K, 1, host, N, K, K, y.data_ptr(), N, 0, s, rows, ks, grid)
        e1.record(); torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    L.host_free(host)
    return best

for N, K in [(1536, 2048), (8192, 4096), (16384, 4096)]:
    for cfg in [(2, 0, 0), (2, 8, 0), (2, 8, 148 * 2), (-1, 0, 0), (-1, 0, 296)]:
        print(json.dumps({"N": N, "K": K, "cfg": cfg, "zero_copy_GBps": round(run(N, K, *cfg), 2)}), flush=True)
