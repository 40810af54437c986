"""Causal varlen prefill attention: tcgen05 kernel (ps_attn_prefill_tc) vs the
mma.sync one (ps_attn_prefill) on BASELINE prefill shapes. CUDA-graph replay of 5
launches, best of 3; TFLOP/s on the causal work (2 * 2 * sum over queries of keys
attended * heads * head_dim)."""
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_26334_b200.runtime import lib as L

SHAPES = [("L8 prefill 2048", 32, 8, 128, [(0, 2048)]),
          ("L8 batched 32 x 512", 32, 8, 128, [(0, 512)] * 32),
          ("L70 prefill 4096", 64, 8, 128, [(0, 4096)]),
          ("Q30 prefill 1024", 32, 4, 128, [(0, 1024)]),
          ("L8 chunk 512 @ 8192", 32, 8, 128, [(8192, 512)])]


def run(kernel, h, kv, hd, seqs):
    torch.manual_seed(0)   # both kernels see the same inputs
    B = len(seqs)
    cap = max(p + n for p, n in seqs)
    pps = -(-cap // 64)                    # paged cache: request b owns pages [b * pps, (b + 1) * pps)
    cache = torch.randn(B * pps * 64, 2, kv, hd, device="cuda").to(torch.bfloat16)
    bt = torch.arange(B * pps, dtype=torch.int32, device="cuda").view(B, pps)
    T = sum(n for _, n in seqs)
    q = torch.randn(T, (h + 2 * kv) * hd, device="cuda")
    qs = torch.tensor(np.cumsum([0] + [n for _, n in seqs]).astype(np.int32), device="cuda")
    p0 = torch.tensor([p for p, _ in seqs], dtype=torch.int32, device="cuda")
    out = torch.empty(T, h * hd, device="cuda", dtype=torch.bfloat16)
    ldq = (h + 2 * kv) * hd

    def launch():
        s = torch.cuda.current_stream().cuda_stream
        if kernel == "tc":
            L.call("ps_attn_prefill_tc", q.data_ptr(), ldq, B, qs.data_ptr(), p0.data_ptr(), 0,
                   max(n for _, n in seqs), h, kv, hd, cache.data_ptr(), 2 * kv * hd, bt.data_ptr(), pps, 64,
                   B * pps, 1 / math.sqrt(hd), out.data_ptr(), h * hd, 1, s)
        else:
            L.call("ps_attn_prefill", q.data_ptr(), ldq, B, qs.data_ptr(), p0.data_ptr(), 0,
                   max(n for _, n in seqs), h, kv, hd, cache.data_ptr(), 2 * kv * hd, bt.data_ptr(), pps, 64,
                   1 / math.sqrt(hd), out.data_ptr(), h * hd, 1, s)
    launch(); launch(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(5):
            launch()
    g.replay(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 5 / 1e3)
    attended = sum(sum(p + i + 1 for i in range(n)) for p, n in seqs)
    flops = 4.0 * attended * h * hd
    return best, flops / best / 1e12, out.float().clone()


for name, h, kv, hd, seqs in SHAPES:
    t_tc, tf_tc, o_tc = run("tc", h, kv, hd, seqs)
    t_hm, tf_hm, o_hm = run("hmma", h, kv, hd, seqs)
    diff = float((o_tc - o_hm).abs().max() / o_hm.abs().max())
    print(json.dumps({"shape": name, "tc_us": round(t_tc * 1e6, 1), "tc_tflops": round(tf_tc, 1),
                      "mma_sync_us": round(t_hm * 1e6, 1), "mma_sync_tflops": round(tf_hm, 1),
                      "speedup": round(t_hm / t_tc, 2), "max_rel_diff": diff}), flush=True)
