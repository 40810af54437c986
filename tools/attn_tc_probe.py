import sys, math, ctypes
sys.path.insert(0, ".")
import numpy as np, torch
from paper_2604_26334_b200.runtime import lib as L
for hd, h, kv, seqs in [(64, 8, 8, [(0, 128)]), (128, 32, 8, [(0, 128)]), (128, 32, 8, [(0, 300)])]:
    B = len(seqs); cap = max(p0 + n for p0, n in seqs)
    cache = torch.randn(cap, B, 2, kv, hd, device="cuda").to(torch.bfloat16)
    T = sum(n for _, n in seqs)
    q = torch.randn(T, h * hd, device="cuda")
    qs = torch.tensor(np.cumsum([0] + [n for _, n in seqs]).astype(np.int32), device="cuda")
    p0 = torch.tensor([p for p, _ in seqs], dtype=torch.int32, device="cuda")
    out = torch.zeros(T, h * hd, device="cuda", dtype=torch.bfloat16)
    L.call("ps_attn_prefill_tc", q.data_ptr(), h * hd, B, qs.data_ptr(), p0.data_ptr(), 0, max(n for _, n in seqs), h, kv, hd,
           cache.data_ptr(), 2 * kv * hd, B * 2 * kv * hd, cap, 1 / math.sqrt(hd), out.data_ptr(), h * hd, 1,
           torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    code = ctypes.c_uint()
    L.call("ps_attn_tc_watchdog", ctypes.byref(code), 1)
    # reference (causal)
    n = seqs[0][1]; s0 = seqs[0][0]
    K = cache[: s0 + n, 0, 0].float(); V = cache[: s0 + n, 0, 1].float()
    G = h // kv
    qq = q[:n].view(n, h, hd)
    Kr = K.repeat_interleave(G, dim=1); Vr = V.repeat_interleave(G, dim=1)
    sc = torch.einsum("thd,shd->hts", qq, Kr) / math.sqrt(hd)
    pos = torch.arange(s0, s0 + n, device="cuda")
    mask = torch.arange(s0 + n, device="cuda")[None, :] > pos[:, None]
    sc = sc.masked_fill(mask[None], float("-inf"))
    ref = torch.einsum("hts,shd->thd", torch.softmax(sc, -1), Vr)
    err = float((out[:n].float().view(n, h, hd) - ref).abs().max() / ref.abs().max())
    print(hd, h, kv, seqs, "watchdog", hex(code.value), "rel err", err, flush=True)
