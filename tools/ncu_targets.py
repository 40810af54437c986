"""One kernel configuration launched `reps` times, for `ncu --set full -k regex:<name> -s 2 -c 1`
captures (round-2 evidence: profiles/r02_ncu_*). Usage: python tools/ncu_targets.py <target>

targets: gemv_bf16 | gemv_coded (28672 x 4096, t = 1, SwiGLU: the bench's kernel_roofline
matrix), gemv_tc_bf16 | gemv_tc_coded (same matrix, t = 32), moe_coded (Qwen3-30B-A3B
one-token experts, k = 8, coded), attn_tc (Llama-3.3-70B 4096-token causal prefill over a
paged cache), expand (8192 x 4096 coded piece -> bf16), hx_expand (one 32 MB run of the
235 MB matrix, Huffman-coded -> bf16), rmsnorm_vec (16384 x 4096 GEMM-pass RMSNorm to bf16)."""
import ctypes
import math
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.runtime import lib as L, wcomp  # noqa: E402

target = sys.argv[1]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 4
s = torch.cuda.current_stream().cuda_stream
g = torch.Generator(device="cuda").manual_seed(0)


def mat(N, K):
    W = ((torch.rand(N, K, device="cuda", generator=g) * 2 - 1) * math.sqrt(3 / K)).to(torch.bfloat16)
    coded, _ = wcomp.encode(W.view(torch.int16).cpu().numpy().view(np.uint16))
    return W, torch.from_numpy(coded).cuda(), coded.shape[1]


if target.startswith("gemv"):
    N, K = 28672, 4096
    W, Wc, rb = mat(N, K)
    t = 32 if "_tc_" in target else 1
    x = torch.randn(t, K, device="cuda")
    y = torch.zeros(t, N // 2, device="cuda")
    ws_n = ctypes.c_longlong()
    L.call("ps_gemv_tc_workspace", N, K, ctypes.byref(ws_n))
    ws = torch.empty(ws_n.value, dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        if target == "gemv_bf16":
            L.call("ps_gemv_bf16", x.data_ptr(), K, 1, W.data_ptr(), N, K, K, y.data_ptr(), N // 2, 2, s)
        elif target == "gemv_coded":
            L.call("ps_gemv_bf16c", x.data_ptr(), K, 1, Wc.data_ptr(), N, K, rb, y.data_ptr(), N // 2, 2, s)
        elif target == "gemv_tc_bf16":
            L.call("ps_gemv_tc", x.data_ptr(), K, t, W.data_ptr(), N, K, K, 0, y.data_ptr(), N // 2, 2,
                   ws.data_ptr(), ws.numel(), s)
        else:
            L.call("ps_gemv_tc", x.data_ptr(), K, t, Wc.data_ptr(), N, K, rb, 1, y.data_ptr(), N // 2, 2,
                   ws.data_ptr(), ws.numel(), s)
elif target == "expand":
    N, K = 8192, 4096
    W, Wc, rb = mat(N, K)
    out = torch.empty(N, K, dtype=torch.bfloat16, device="cuda")
    for _ in range(reps):
        L.call("ps_expand_coded", Wc.data_ptr(), rb, N, K, out.data_ptr(), K, s)
    torch.cuda.synchronize()
    assert torch.equal(out, W)
elif target == "hx_expand":   # the 235 MB matrix, Huffman-coded, expanded in 32 MB runs (decode pass)
    from paper_2604_26334_b200.runtime import hxcodec as hx
    N, K = 28672, 4096
    W = ((torch.rand(N, K, device="cuda", generator=g) * 2 - 1) * math.sqrt(3 / K)).to(torch.bfloat16)
    enc = hx.GpuHxEncoder()
    fill = lambda dst, r0, r1: L.memcpy_async(dst, W.data_ptr() + r0 * K * 2, (r1 - r0) * K * 2, s)  # noqa: E731
    m = enc.plan(fill, N, K)
    host = L.host_alloc(m.nbytes, mapped=False)
    enc.write(fill, m, host)
    blob = torch.empty(m.nbytes, dtype=torch.uint8, device="cuda")
    L.memcpy_async(blob.data_ptr(), host, m.nbytes, s)
    torch.cuda.synchronize()
    lut = torch.from_numpy(m.lut.view(np.int32)).cuda()
    out = torch.empty(N, K, dtype=torch.bfloat16, device="cuda")
    rr = (32 << 20) // (K * 2)
    rel = torch.from_numpy((m.block_off[:rr // 64] - m.block_off[0]).astype(np.int32)).cuda()
    for _ in range(reps):
        L.call("ps_hx_expand", blob.data_ptr(), rel.data_ptr(), rr, K, lut.data_ptr(), out.data_ptr(), K, s)
    torch.cuda.synchronize()
    assert torch.equal(out[:rr], W[:rr])
elif target == "moe_coded":
    E, k, d, eff = 32, 8, 2048, 768
    gu = [mat(2 * eff, d) for _ in range(E)]
    dn = [mat(d, eff) for _ in range(E)]
    tg, td = max(c[2] for c in gu) - d * 3 // 2, max(c[2] for c in dn) - eff * 3 // 2
    up = lambda n: (n + 255) // 256 * 256  # noqa: E731
    gu_rb, d_rb = wcomp.row_bytes(d, tg), wcomp.row_bytes(eff, td)
    down_off = up(2 * eff * gu_rb)
    stride = up(down_off + d * d_rb)
    blob = np.zeros(E * stride, np.uint8)
    for e in range(E):
        wcomp.encode(gu[e][0].view(torch.int16).cpu().numpy().view(np.uint16), out=blob[e * stride:], trailer=tg)
        wcomp.encode(dn[e][0].view(torch.int16).cpu().numpy().view(np.uint16), out=blob[e * stride + down_off:],
                     trailer=td)
    cb = torch.from_numpy(blob).cuda()
    ids = torch.arange(0, 2 * k, 2, dtype=torch.int32, device="cuda")
    w = torch.rand(k, device="cuda")
    x = torch.randn(1, d, device="cuda")
    h = torch.zeros(k, eff, device="cuda")
    y = torch.zeros(1, d, device="cuda")
    for _ in range(reps):
        L.call("ps_moe_decode_experts_c", x.data_ptr(), ids.data_ptr(), k, None, cb.data_ptr(), stride, 0, down_off,
               eff, d, gu_rb, d_rb, h.data_ptr(), w.data_ptr(), y.data_ptr(), s)
elif target == "attn_tc":
    h, kv, hd, n = 64, 8, 128, 4096
    pps = n // 64
    perm = torch.tensor(np.random.default_rng(0).permutation(pps).astype(np.int32), device="cuda").view(1, pps)
    pool = torch.randn(n, 2 * kv * hd, device="cuda").to(torch.bfloat16)
    q = torch.randn(n, (h + 2 * kv) * hd, device="cuda")
    qs = torch.tensor([0, n], dtype=torch.int32, device="cuda")
    p0 = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = torch.empty(n, h * hd, device="cuda", dtype=torch.bfloat16)
    for _ in range(reps):
        L.call("ps_attn_prefill_tc", q.data_ptr(), (h + 2 * kv) * hd, 1, qs.data_ptr(), p0.data_ptr(), 0, n, h, kv,
               hd, pool.data_ptr(), 2 * kv * hd, perm.data_ptr(), pps, 64, pps, 1 / math.sqrt(hd), out.data_ptr(),
               h * hd, 1, s)
elif target == "rmsnorm_vec":   # the config-4 prefill shape: 16384 rows x 4096, fp32 -> bf16
    n, d = 16384, 4096
    x = torch.randn(n, d, device="cuda")
    w = torch.ones(d, device="cuda").to(torch.bfloat16)
    o = torch.empty(n, d, device="cuda", dtype=torch.bfloat16)
    for _ in range(reps):
        L.call("ps_rmsnorm", x.data_ptr(), d, None, n, w.data_ptr(), d, 1e-5, o.data_ptr(), d, 1, s)
else:
    raise SystemExit(f"unknown target {target}")
torch.cuda.synchronize()
print("ok", target)
