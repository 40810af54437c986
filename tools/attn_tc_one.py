"""One L70-shaped causal prefill (4096 tokens, 64 heads / 8 kv, hd 128) through
ps_attn_prefill_tc, launched 3 times, for ncu captures."""
import math, sys
import numpy as np, torch
sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L
h, kv, hd, n = 64, 8, 128, 4096
cache = torch.randn(n, 1, 2, kv, hd, device="cuda").to(torch.bfloat16)   # paged: pages 0.. in order
bt = torch.arange(n // 64, dtype=torch.int32, device="cuda").view(1, -1)
q = torch.randn(n, h * hd, device="cuda")
qs = torch.tensor([0, n], dtype=torch.int32, device="cuda"); p0 = torch.zeros(1, dtype=torch.int32, device="cuda")
out = torch.empty(n, h * hd, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    L.call("ps_attn_prefill_tc", q.data_ptr(), h * hd, 1, qs.data_ptr(), p0.data_ptr(), 0, n, h, kv, hd,
           cache.data_ptr(), 2 * kv * hd, bt.data_ptr(), n // 64, 64, n // 64, 1 / math.sqrt(hd), out.data_ptr(), h * hd, 1,
           torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
