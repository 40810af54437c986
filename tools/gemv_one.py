"""One GEMV shape launched 4 times (L2 flushed between) for ncu captures:
python tools/gemv_one.py N K [t] [rows] [epi]  (rows 0 = bulk-copy kernel, 2 = register-burst;
epi 0 store, 1 accumulate, 2 SwiGLU)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L

N, K = int(sys.argv[1]), int(sys.argv[2])
t = int(sys.argv[3]) if len(sys.argv) > 3 else 1
rows = int(sys.argv[4]) if len(sys.argv) > 4 else 0
epi = int(sys.argv[5]) if len(sys.argv) > 5 else 0
W = torch.empty(N, K, dtype=torch.bfloat16, device="cuda").normal_()
x = torch.randn(t, K, device="cuda")
ldy = N // 2 if epi == 2 else N
y = torch.zeros(t, ldy, device="cuda")
flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB > L2
s = torch.cuda.current_stream().cuda_stream
for i in range(4):
    flush.sum()
    L.call("ps_gemv_bf16_cfg", x.data_ptr(), K, t, W.data_ptr(), N, K, K, y.data_ptr(), ldy, epi, s, rows, 0, 0)
torch.cuda.synchronize()
