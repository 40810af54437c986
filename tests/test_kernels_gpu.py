"""Per-kernel parity on the B200, through the C-ABI (include/pshard.h).

Each kernel is compared with a plain fp32 PyTorch restatement on the same
inputs. Tolerances: fp32-accumulated kernels on fp32 activations must agree
to ~1e-5 relative; kernels that take bf16 activations (tcgen05 GEMM,
mma.sync flash attention) are bounded by bf16 input rounding (2^-8).
Integer work (argmax, weight init) must be bit-exact.
"""

import ctypes as C
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def L():
    from paper_2604_26334_b200.runtime import lib
    return lib


def stream():
    return torch.cuda.current_stream().cuda_stream


def rel_err(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


@pytest.mark.parametrize("t", [1, 2, 3, 4, 8, 13, 32])
@pytest.mark.parametrize("epi", [0, 1, 2])
@pytest.mark.parametrize("N,K", [(6144, 4096), (256, 14336), (130, 512), (28672, 4096), (4096, 14336),
                                 (1000, 1544), (2, 2056)])
@pytest.mark.parametrize("rows", [0, 2])
def test_gemv(t, epi, N, K, rows):
    """rows 0 = bulk-copy kernel (gemv_tma.cu), 2 = register-burst kernel (gemv.cu).
    Shapes cover partial K chunks (1544, 2056 = 2048 + 8), odd row counts per CTA
    and a matrix with fewer rows than SMs."""
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(t * 100 + N)
    x = torch.randn(t, K, device="cuda", generator=g)
    W = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    ref = x @ W.float().T
    if epi == 2:
        ref = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
        y = torch.zeros(t, N // 2, device="cuda")
        ldy = N // 2
    else:
        y = torch.randn(t, N, device="cuda", generator=g) if epi == 1 else torch.zeros(t, N, device="cuda")
        if epi == 1:
            ref = ref + y
        ldy = N
    lib.call("ps_gemv_bf16_cfg", x.data_ptr(), K, t, W.data_ptr(), N, K, K, y.data_ptr(), ldy, epi, stream(),
             rows, 0, 0)
    torch.cuda.synchronize()
    assert rel_err(y, ref) < 2e-5


def test_gemv_zero_copy_host_weights():
    lib = L()
    N, K = 512, 4096
    W = (torch.randn(N, K) / 64).to(torch.bfloat16)
    host = lib.host_alloc(W.numel() * 2, mapped=True)
    import ctypes
    ctypes.memmove(host, W.data_ptr(), W.numel() * 2)
    x = torch.randn(1, K, device="cuda")
    y = torch.zeros(1, N, device="cuda")
    lib.call("ps_gemv_bf16", x.data_ptr(), K, 1, host, N, K, K, y.data_ptr(), N, 0, stream())
    torch.cuda.synchronize()
    assert rel_err(y, x @ W.float().cuda().T) < 2e-5
    lib.host_free(host)


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (2048, 6144, 4096), (200, 1000, 512),
                                   (4096, 512, 14336), (64, 256, 1536), (16384, 768, 512),
                                   (300, 28672, 256), (1, 256, 64), (257, 130, 128)])
@pytest.mark.parametrize("epi", [0, 1, 3, 2])
@pytest.mark.parametrize("variant", [0, 1, 2])
def test_gemm_tcgen05(M, N, K, epi, variant):
    """variant 0 = auto, 1 = one 128x256 tile per CTA, 2 = persistent CTA-pair
    (cta_group::2) kernel; the pair kernel's tails (M or N not a tile multiple,
    a pair whose second CTA is entirely out of bounds) are covered."""
    if variant == 1 and M > 4096:
        pytest.skip("1-CTA kernel: covered at smaller M")
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda", generator=g) / math.sqrt(K)).to(torch.bfloat16)
    ref = A.float() @ B.float().T
    if epi == 2:
        ref = torch.nn.functional.silu(ref[:, 0::2]) * ref[:, 1::2]
        C = torch.zeros(M, N // 2, device="cuda", dtype=torch.bfloat16)
        ldc = N // 2
    elif epi == 3:
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
        ldc = N
    else:
        C = torch.randn(M, N, device="cuda", generator=g) if epi == 1 else torch.zeros(M, N, device="cuda")
        if epi == 1:
            ref = ref + C
        ldc = N
    lib.call("ps_gemm_bf16_cfg", A.data_ptr(), M, K, K, B.data_ptr(), N, K, C.data_ptr(), ldc, epi,
             stream(), variant)
    torch.cuda.synchronize()
    tol = 4e-5 if epi in (0, 1) else 8e-3   # fp32 accumulation order / bf16 output rounding
    assert rel_err(C.float(), ref) < tol


def test_rmsnorm_rows_and_bf16():
    lib = L()
    x = torch.randn(5, 4096, device="cuda")
    w = (1 + 0.1 * torch.randn(4096, device="cuda")).to(torch.bfloat16)
    rows = torch.tensor([4, 0, 2], dtype=torch.int32, device="cuda")
    out = torch.zeros(3, 4096, device="cuda")
    lib.call("ps_rmsnorm", x.data_ptr(), 4096, rows.data_ptr(), 3, w.data_ptr(), 4096, 1e-5,
             out.data_ptr(), 4096, 0, stream())
    xs = x[rows.long()]
    ref = xs * torch.rsqrt(xs.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    torch.cuda.synchronize()
    assert rel_err(out, ref) < 1e-5
    o16 = torch.zeros(5, 4096, device="cuda", dtype=torch.bfloat16)
    lib.call("ps_rmsnorm", x.data_ptr(), 4096, 0, 5, w.data_ptr(), 4096, 1e-5, o16.data_ptr(), 4096, 1, stream())
    ref5 = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    torch.cuda.synchronize()
    assert rel_err(o16.float(), ref5) < 8e-3


@pytest.mark.parametrize("n,d,ldx,gather", [(300, 4096, 4096, False), (257, 5120, 5128, True), (64, 8192, 8192, False),
                                             (100, 2048, 2048, True)])
def test_rmsnorm_bf16_many_rows(n, d, ldx, gather):
    """GEMM-pass RMSNorm to bf16 (>= 64 rows: the vectorised kernel): within bf16 rounding
    of the fp32 reference, every element; the row-gather form too."""
    lib = L()
    x = torch.randn(n, ldx, device="cuda")
    w = (1 + 0.1 * torch.randn(d, device="cuda")).to(torch.bfloat16)
    rows = torch.randperm(n, device="cuda").to(torch.int32) if gather else None
    o16 = torch.zeros(n, d + 8, device="cuda", dtype=torch.bfloat16)
    lib.call("ps_rmsnorm", x.data_ptr(), ldx, rows.data_ptr() if gather else 0, n, w.data_ptr(), d, 1e-5,
             o16.data_ptr(), d + 8, 1, stream())
    xs = (x[rows.long()] if gather else x)[:, :d]
    ref = xs * torch.rsqrt(xs.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    torch.cuda.synchronize()
    got = o16[:, :d].float()
    assert torch.all((got - ref).abs() <= ref.abs() * 2 ** -8 + 1e-6)
    assert torch.all(o16[:, d:] == 0)


def _rope_ref(x, pos, inv):
    hd = x.shape[-1]
    ang = pos.double()[:, None] * inv[None, :].double()
    cos, sin = torch.cos(ang).float()[:, None, :], torch.sin(ang).float()[:, None, :]
    a, b = x[..., : hd // 2], x[..., hd // 2:]
    return torch.cat([a * cos - b * sin, b * cos + a * sin], -1)


PAGE = 64


def paged(dense, lens, page_rows=PAGE, seed=0, spare=3):
    """Dense per-request rows [cap, B, ...] -> (pool [pages * page_rows, row], block table
    [B, pages per slot] int32) with the pages of all requests SHUFFLED over a pool with
    `spare` unused pages; every row a request does not own (unused pages, rows past its
    length) holds NaN, so a kernel that reads one is caught."""
    cap, B = dense.shape[0], dense.shape[1]
    row = dense[0, 0].numel()
    pps = -(-cap // page_rows)
    need = [-(-n // page_rows) for n in lens]
    n_pages = sum(need) + spare
    perm = np.random.default_rng(seed).permutation(n_pages)
    pool = torch.full((n_pages * page_rows, row), float("nan"), device=dense.device).to(dense.dtype)
    table = np.full((B, pps), -1, np.int32)
    k = 0
    for b, n in enumerate(lens):
        for j in range(need[b]):
            pg = int(perm[k]); k += 1
            table[b, j] = pg
            r0, r1 = j * page_rows, min(n, (j + 1) * page_rows)
            pool[pg * page_rows:pg * page_rows + (r1 - r0)] = dense[r0:r1, b].reshape(r1 - r0, row)
    return pool, torch.from_numpy(table).to(dense.device), n_pages


@pytest.mark.parametrize("hd,h,kv,qk", [(128, 32, 8, False), (64, 8, 8, False), (128, 32, 4, True)])
def test_qkv_rope_append(hd, h, kv, qk):
    lib = L()
    T, B, cap = 6, 3, 40
    rows = (h + 2 * kv) * hd
    qkv = torch.randn(T, rows, device="cuda")
    pos = torch.tensor([3, 4, 5, 0, 9, 10], dtype=torch.int32, device="cuda")
    req = torch.tensor([2, 2, 2, 0, 1, 1], dtype=torch.int32, device="cuda")
    inv = 1.0 / (10000.0 ** (torch.arange(0, hd, 2, dtype=torch.float64) / hd))
    ang = torch.arange(cap, dtype=torch.float64)[:, None] * inv[None, :]
    rope = torch.stack([torch.cos(ang), torch.sin(ang)], -1).float().cuda()
    # paged cache: request slot b owns pages table[b] (shuffled, 2 per slot)
    pps = -(-cap // PAGE)
    table = torch.tensor(np.random.default_rng(hd + h).permutation(B * pps).reshape(B, pps).astype(np.int32),
                         device="cuda")
    pool = torch.zeros(B * pps * PAGE, 2 * kv * hd, dtype=torch.bfloat16, device="cuda")
    qn = (1 + 0.1 * torch.randn(hd, device="cuda")).to(torch.bfloat16) if qk else None
    kn = (1 + 0.1 * torch.randn(hd, device="cuda")).to(torch.bfloat16) if qk else None
    src = qkv.clone()
    lib.call("ps_qkv_rope_append", qkv.data_ptr(), rows, T, h, kv, hd, pos.data_ptr(), req.data_ptr(),
             pool.data_ptr(), 2 * kv * hd, table.data_ptr(), pps, PAGE, rope.data_ptr(),
             qn.data_ptr() if qk else 0, kn.data_ptr() if qk else 0, 1e-6, stream())
    torch.cuda.synchronize()
    q = src[:, : h * hd].view(T, h, hd)
    k = src[:, h * hd:(h + kv) * hd].view(T, kv, hd)
    v = src[:, (h + kv) * hd:].view(T, kv, hd)
    if qk:
        q = q * torch.rsqrt(q.pow(2).mean(-1, keepdim=True) + 1e-6) * qn.float()
        k = k * torch.rsqrt(k.pow(2).mean(-1, keepdim=True) + 1e-6) * kn.float()
    q = _rope_ref(q.cpu(), pos.cpu(), inv).cuda()
    k = _rope_ref(k.cpu(), pos.cpu(), inv).cuda()
    assert rel_err(qkv[:, : h * hd].view(T, h, hd), q) < 1e-5
    for t in range(T):
        p, b = int(pos[t]), int(req[t])
        row = pool[int(table[b, p // PAGE]) * PAGE + p % PAGE].float()
        assert rel_err(row[: kv * hd].view(kv, hd), k[t]) < 8e-3
        assert rel_err(row[kv * hd:].view(kv, hd), v[t]) < 8e-3


def _attn_ref(q, K, V, qpos):
    # q [T, h, hd]; K, V [S, kvh, hd]
    h, kvh = q.shape[1], K.shape[1]
    G = h // kvh
    Kr, Vr = K.repeat_interleave(G, 1), V.repeat_interleave(G, 1)
    s = torch.einsum("thd,shd->hts", q, Kr) / math.sqrt(q.shape[-1])
    mask = torch.arange(K.shape[0], device=q.device)[None, :] > qpos[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    return torch.einsum("hts,shd->thd", torch.softmax(s, -1), Vr)


@pytest.mark.parametrize("hd,h,kv,lens", [(128, 32, 8, [2304]), (128, 32, 8, [1, 17, 640, 300]),
                                          (64, 8, 8, [160, 5]), (128, 64, 8, [4224]),
                                          (128, 32, 4, [1000]), (128, 32, 32, [16384, 129]),
                                          (128, 32, 8, [33, 128, 127, 1])])
def test_attn_decode(hd, h, kv, lens):
    """Split-KV decode over a paged cache with shuffled pages (NaN everywhere a request
    does not own): every request's output matches fp32 attention over its own rows."""
    lib = L()
    B, cap = len(lens), max(lens)
    g = torch.Generator(device="cuda").manual_seed(sum(lens))
    cache = torch.randn(cap, B, 2, kv, hd, device="cuda", generator=g).to(torch.bfloat16)
    pool, table, _ = paged(cache, lens, seed=sum(lens))
    q = torch.randn(B, h * hd, device="cuda", generator=g)
    ln = torch.tensor(lens, dtype=torch.int32, device="cuda")
    out = torch.zeros(B, h * hd, device="cuda")
    ws = torch.zeros(max(1, lib.attn_decode_workspace(B, h, hd, cap)), device="cuda")
    lib.call("ps_attn_decode", q.data_ptr(), h * hd, B, h, kv, hd, 0, pool.data_ptr(), 2 * kv * hd,
             table.data_ptr(), table.shape[1], PAGE, ln.data_ptr(), cap, 1 / math.sqrt(hd), out.data_ptr(), h * hd,
             ws.data_ptr(), ws.numel(), stream())
    torch.cuda.synchronize()
    for b, n in enumerate(lens):
        K = cache[:n, b, 0].float()
        V = cache[:n, b, 1].float()
        ref = _attn_ref(q[b].view(1, h, hd), K, V, torch.tensor([n - 1], device="cuda"))
        assert rel_err(out[b].view(1, h, hd), ref) < 1e-4


@pytest.mark.parametrize("hd,h,kv,seqs", [(128, 32, 8, [(0, 2048)]), (64, 8, 8, [(0, 128)]),
                                          (128, 32, 8, [(0, 100), (37, 64), (500, 5)]),
                                          (128, 32, 4, [(0, 300)]), (128, 64, 8, [(3000, 200)]),
                                          (128, 32, 8, [(0, 512)] * 4), (64, 4, 2, [(7, 129), (0, 1)])])
@pytest.mark.parametrize("kernel", ["ps_attn_prefill", "ps_attn_prefill_tc"])
def test_attn_prefill(hd, h, kv, seqs, kernel):
    """kernel: the mma.sync flash attention or the tcgen05/TMEM/TMA one; varlen
    requests with p0 > 0 (chunked prefill), GQA groups 1-8, head dims 64 / 128,
    partial query and key blocks; paged cache with shuffled pages and NaN in every row a
    request does not own (its last page's tail included)."""
    lib = L()
    B = len(seqs)
    cap = max(p0 + n for p0, n in seqs)
    g = torch.Generator(device="cuda").manual_seed(cap + B)
    cache = torch.randn(cap, B, 2, kv, hd, device="cuda", generator=g).to(torch.bfloat16)
    pool, table, n_pages = paged(cache, [p0 + n for p0, n in seqs], seed=cap)
    T = sum(n for _, n in seqs)
    q = torch.randn(T, h * hd, device="cuda", generator=g)
    q_start = np.cumsum([0] + [n for _, n in seqs]).astype(np.int32)
    qs = torch.tensor(q_start, device="cuda")
    p0 = torch.tensor([p for p, _ in seqs], dtype=torch.int32, device="cuda")
    out = torch.zeros(T, h * hd, device="cuda", dtype=torch.bfloat16)
    if kernel == "ps_attn_prefill":
        lib.call("ps_attn_prefill", q.data_ptr(), h * hd, B, qs.data_ptr(), p0.data_ptr(), 0,
                 max(n for _, n in seqs), h, kv, hd, pool.data_ptr(), 2 * kv * hd, table.data_ptr(),
                 table.shape[1], PAGE, 1 / math.sqrt(hd), out.data_ptr(), h * hd, 1, stream())
    else:
        lib.call("ps_attn_prefill_tc", q.data_ptr(), h * hd, B, qs.data_ptr(), p0.data_ptr(), 0,
                 max(n for _, n in seqs), h, kv, hd, pool.data_ptr(), 2 * kv * hd, table.data_ptr(),
                 table.shape[1], PAGE, n_pages, 1 / math.sqrt(hd), out.data_ptr(), h * hd, 1, stream())
    torch.cuda.synchronize()
    for b, (s0, n) in enumerate(seqs):
        K = cache[: s0 + n, b, 0].float()
        V = cache[: s0 + n, b, 1].float()
        qb = q[q_start[b]:q_start[b] + n].view(n, h, hd)
        ref = _attn_ref(qb, K, V, torch.arange(s0, s0 + n, device="cuda"))
        assert rel_err(out[q_start[b]:q_start[b] + n].float().view(n, h, hd), ref) < 2e-2


def test_argmax_ties_lowest_index():
    lib = L()
    x = torch.randn(4, 128256, device="cuda")
    x[1, 77] = 1e9
    x[1, 5000] = 1e9
    out = torch.zeros(4, dtype=torch.int32, device="cuda")
    lib.call("ps_argmax", x.data_ptr(), 4, 128256, 128256, out.data_ptr(), stream())
    torch.cuda.synchronize()
    assert out.tolist() == torch.argmax(x, -1).int().tolist()
    assert out[1].item() == 77


def test_embed_gather_zero_copy():
    lib = L()
    V, d = 1000, 512
    table = torch.randn(V, d).to(torch.bfloat16)
    host = lib.host_alloc(V * d * 2, mapped=True)
    import ctypes
    ctypes.memmove(host, table.data_ptr(), V * d * 2)
    ids = torch.tensor([5, 999, 0], dtype=torch.int32, device="cuda")
    out = torch.zeros(3, d, device="cuda")
    lib.call("ps_embed_gather", host, ids.data_ptr(), 3, d, out.data_ptr(), d, stream())
    torch.cuda.synchronize()
    assert torch.equal(out.cpu(), table[ids.cpu().long()].float())
    lib.host_free(host)


def test_upload_small():
    lib = L()
    arr = np.arange(1000, dtype=np.int32)
    dst = torch.zeros(1000, dtype=torch.int32, device="cuda")
    lib.call("ps_upload_small", dst.data_ptr(), arr.ctypes.data, arr.nbytes, stream())
    torch.cuda.synchronize()
    assert dst.cpu().numpy().tolist() == arr.tolist()


def test_weight_init_bit_exact_vs_oracle():
    from oracle import model_ref
    lib = L()
    n_rows, cols = 300, 4096
    buf = torch.zeros(n_rows * cols, dtype=torch.int16, device="cuda")
    sd = model_ref.seed_of(3, "L1.wo")
    sc, bi = model_ref.scale_bias("L1.wo", cols)
    # generate in two chunks to exercise the offset argument
    half = (n_rows // 2) * cols
    lib.call("ps_init_uniform_bf16", buf.data_ptr(), half, sd, 0, sc, bi, stream())
    lib.call("ps_init_uniform_bf16", buf.data_ptr() + half * 2, n_rows * cols - half, sd, half, sc, bi, stream())
    torch.cuda.synchronize()
    got = buf.cpu().numpy().view(np.uint16).reshape(n_rows, cols)
    np.testing.assert_array_equal(got, model_ref.bf16_bits(3, "L1.wo", n_rows, cols))
    gu = torch.zeros(2 * 50 * cols, dtype=torch.int16, device="cuda")
    sa, sb = model_ref.seed_of(3, "L1.w_gate"), model_ref.seed_of(3, "L1.w_up")
    sc, bi = model_ref.scale_bias("L1.w_gate", cols)
    lib.call("ps_init_interleaved_bf16", gu.data_ptr(), 50, 0, 37, cols, sa, sb, sc, bi, stream())
    lib.call("ps_init_interleaved_bf16", gu.data_ptr() + 37 * cols * 2, 50, 37, 63, cols, sa, sb, sc, bi, stream())
    torch.cuda.synchronize()
    got = gu.cpu().numpy().view(np.uint16).reshape(100, cols)
    np.testing.assert_array_equal(got, model_ref.interleaved_bits(3, "L1.w_gate", "L1.w_up", 50, cols))


def _moe_ref(x, router, Wgu, Wd, k):
    """fp32 Qwen3-MoE block: softmax, top-k, renormalise, SwiGLU experts."""
    probs = torch.softmax(x @ router.T, -1)
    w, ids = torch.topk(probs, k, -1)
    w = w / w.sum(-1, keepdim=True)
    out = torch.zeros_like(x)
    for t in range(x.shape[0]):
        for j in range(k):
            e = int(ids[t, j])
            gu = Wgu[e] @ x[t]
            h = torch.nn.functional.silu(gu[0::2]) * gu[1::2]
            out[t] += w[t, j] * (Wd[e] @ h)
    return out, ids, w


@pytest.mark.parametrize("T,zero_copy,x_bf16", [(1, True, False), (3, False, False), (40, False, True)])
def test_moe_pipeline(T, zero_copy, x_bf16):
    lib = L()
    E, k, d, eff = 16, 4, 256, 128
    g = torch.Generator(device="cuda").manual_seed(T)
    x = torch.randn(T, d, device="cuda", generator=g)
    router = (torch.randn(E, d, device="cuda", generator=g) / 8).to(torch.bfloat16)
    Wgu = (torch.randn(E, 2 * eff, d, device="cuda", generator=g) / 16).to(torch.bfloat16)
    Wd = (torch.randn(E, d, eff, device="cuda", generator=g) / 11).to(torch.bfloat16)
    # expert blob: [wgu_e | wdown_e] per expert
    blob = torch.cat([torch.cat([Wgu[e].reshape(-1), Wd[e].reshape(-1)]) for e in range(E)]).contiguous()
    stride = (2 * eff * d + d * eff) * 2
    base = blob.data_ptr()
    host = None
    if zero_copy:
        import ctypes
        host = lib.host_alloc(blob.numel() * 2, mapped=True)
        cpu = blob.cpu()
        ctypes.memmove(host, cpu.data_ptr(), blob.numel() * 2)
        base = host
    s = stream()
    xin = x.to(torch.bfloat16) if x_bf16 else x
    logits = xin.float() @ router.float().T
    P = T * k
    ids = torch.zeros(P, dtype=torch.int32, device="cuda")
    w = torch.zeros(P, device="cuda")
    import ctypes
    n = ctypes.c_longlong()
    lib.call("ps_moe_plan_ints", P, E, ctypes.byref(n))
    plan = torch.zeros(n.value, dtype=torch.int32, device="cuda")
    h = torch.zeros(P, eff, device="cuda")
    out = torch.zeros(P, d, device="cuda")
    y = torch.randn(T, d, device="cuda", generator=g)
    y0 = y.clone()
    lib.call("ps_moe_route_topk", logits.data_ptr(), E, T, E, k, 1, ids.data_ptr(), w.data_ptr(), s)
    lib.call("ps_moe_plan", ids.data_ptr(), P, E, plan.data_ptr(), s)
    xin = x.to(torch.bfloat16) if x_bf16 else x
    # process experts in two ranges, as a ring piece split would
    for lo, hi in ((0, 7), (7, E)):
        lib.call("ps_moe_expert_gu", xin.data_ptr(), d, 1 if x_bf16 else 0, plan.data_ptr(), E, P, k,
                 base, stride, 0, eff, d, h.data_ptr(), lo, hi, s)
        lib.call("ps_moe_expert_down", h.data_ptr(), plan.data_ptr(), E, P, base, stride, 2 * eff * d * 2,
                 eff, d, out.data_ptr(), lo, hi, s)
    lib.call("ps_moe_combine", out.data_ptr(), plan.data_ptr(), E, P, w.data_ptr(), T, k, d, y.data_ptr(), d, s)
    torch.cuda.synchronize()
    ref, rid, rw = _moe_ref(xin.float(), router.float(), Wgu.float(), Wd.float(), k)
    assert torch.equal(ids.view(T, k).long(), rid)
    assert rel_err(w.view(T, k), rw) < 1e-5
    assert rel_err(y - y0, ref) < 1e-4
    if host:
        lib.host_free(host)


@pytest.mark.parametrize("E,k,d,eff,mapped", [(16, 4, 256, 128, False), (32, 8, 2048, 768, True),
                                              (8, 2, 512, 1536, False), (128, 8, 2048, 768, False)])
def test_moe_decode_experts_one_token(E, k, d, eff, mapped):
    """ps_moe_decode_experts (t = 1, no plan, combine fused) against the fp32 MoE
    block, with and without a fetcher slot map; bit-identical across runs
    (fixed-order combine)."""
    import ctypes
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(E + d)
    x = torch.randn(1, d, device="cuda", generator=g)
    router = (torch.randn(E, d, device="cuda", generator=g) / 8).to(torch.bfloat16)
    Wgu = (torch.randn(E, 2 * eff, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    Wd = (torch.randn(E, d, eff, device="cuda", generator=g) / eff ** 0.5).to(torch.bfloat16)
    blob = torch.cat([torch.cat([Wgu[e].reshape(-1), Wd[e].reshape(-1)]) for e in range(E)]).contiguous()
    stride = (2 * eff * d + d * eff) * 2
    s = stream()
    logits = x @ router.float().T
    ids = torch.zeros(k, dtype=torch.int32, device="cuda")
    w = torch.zeros(k, device="cuda")
    lib.call("ps_moe_route_topk", logits.data_ptr(), E, 1, E, k, 1, ids.data_ptr(), w.data_ptr(), s)
    torch.cuda.synchronize()
    base, slot_map = blob.data_ptr(), None
    if mapped:   # routed experts copied into k slots in reverse order, as a fetcher could
        slots = torch.zeros(k * stride // 2, dtype=torch.bfloat16, device="cuda")
        smap = torch.full((E,), -1, dtype=torch.int32, device="cuda")
        for j, e in enumerate(ids.tolist()):
            sl = k - 1 - j
            slots[sl * stride // 2:(sl + 1) * stride // 2] = blob[e * stride // 2:(e + 1) * stride // 2]
            smap[e] = sl
        base, slot_map = slots.data_ptr(), smap
    h = torch.zeros(k, eff, device="cuda")
    y0 = torch.randn(1, d, device="cuda", generator=g)
    ys = []
    for _ in range(2):
        y = y0.clone()
        lib.call("ps_moe_decode_experts", x.data_ptr(), ids.data_ptr(), k,
                 slot_map.data_ptr() if slot_map is not None else None, base, stride, 0, 2 * eff * d * 2,
                 eff, d, h.data_ptr(), w.data_ptr(), y.data_ptr(), s)
        torch.cuda.synchronize()
        ys.append(y)
    assert torch.equal(ys[0], ys[1])
    ref, rid, rw = _moe_ref(x, router.float(), Wgu.float(), Wd.float(), k)
    assert torch.equal(ids.view(1, k).long(), rid)
    assert rel_err(ys[0] - y0, ref) < 1e-4


def test_expert_fetcher_publish_copy_wait():
    """ps_moe_publish -> host thread copies the routed experts (ascending id) into
    slots -> ps_wait_flag; mapped expert kernels see expert e at its slot."""
    import ctypes
    lib = L()
    E, k, P, nbytes = 16, 4, 8, 4096
    f = ctypes.c_void_p()
    lib.call("ps_fetcher_create", E, ctypes.byref(f))
    try:
        host = lib.host_alloc(E * nbytes, mapped=True)
        src = (np.arange(E * nbytes, dtype=np.uint32) % 251).astype(np.uint8)
        src.reshape(E, nbytes)[:, 0] = np.arange(E)           # expert id in byte 0
        ctypes.memmove(host, src.ctypes.data, src.nbytes)
        slots = torch.zeros(E * nbytes, dtype=torch.uint8, device="cuda")
        slotmap = torch.zeros(E, dtype=torch.int32, device="cuda")
        for seq, ids in enumerate([[3, 9, 3, 1, 15, 9, 0, 1], [2, 2, 2, 2, 2, 2, 2, 2]], start=1):
            dev_ids = torch.tensor(ids, dtype=torch.int32, device="cuda")
            lib.call("ps_fetcher_submit", f, seq, host, nbytes, nbytes, slots.data_ptr(), nbytes)
            lib.call("ps_moe_publish", f, dev_ids.data_ptr(), P, E, slotmap.data_ptr(), seq, stream())
            lib.call("ps_wait_flag", f, seq, stream())
            torch.cuda.synchronize()
            routed = sorted(set(ids))
            m = slotmap.cpu().numpy()
            for e in range(E):
                assert m[e] == (routed.index(e) if e in routed else -1)
            got = slots.cpu().numpy().reshape(E, nbytes)
            for r, e in enumerate(routed):
                assert np.array_equal(got[r], src.reshape(E, nbytes)[e])
        n, b, err = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int()
        lib.call("ps_fetcher_info", f, None, None, ctypes.byref(n), ctypes.byref(b), ctypes.byref(err))
        assert (n.value, err.value) == (5 + 1, 0)
        dev_err = ctypes.c_uint()
        lib.call("ps_fetcher_device_error", f, ctypes.byref(dev_err))
        assert dev_err.value == 0
        lib.host_free(host)
    finally:
        lib.call("ps_fetcher_destroy", f)


def test_expert_fetcher_speculative_slots():
    """ps_moe_publish_spec: a layer's routed experts already in its prediction set are not
    copied (slot_of_rank points at the prediction slot), misses go to slot = rank, and the
    next layer's predictions are copied behind the flag into the other set; the per-seq
    byte count is misses + predictions."""
    import ctypes
    lib = L()
    E, k, S, nbytes = 16, 4, 2, 4096
    n_slots = k + 2 * S
    f = ctypes.c_void_p()
    lib.call("ps_fetcher_create", E, ctypes.byref(f))
    try:
        host = lib.host_alloc(E * nbytes, mapped=True)
        src = (np.arange(E * nbytes, dtype=np.uint32) % 251).astype(np.uint8).reshape(E, nbytes)
        src[:, 0] = np.arange(E)
        ctypes.memmove(host, src.ctypes.data, src.nbytes)
        slots = torch.zeros(n_slots * nbytes, dtype=torch.uint8, device="cuda")
        slotmap = torch.zeros(E, dtype=torch.int32, device="cuda")
        sor = torch.full((k,), -7, dtype=torch.int32, device="cuda")
        state = torch.full((2 * S,), -1, dtype=torch.int32, device="cuda")
        # (routed ids, set_cur, predictions for the next layer, set_next, expected slot_of_rank, copies)
        layers = [([3, 9, 1, 15], -1, [2, 9], 0, [0, 1, 2, 3], 6),
                  ([9, 2, 5, 6], 0, [7, 8], 1, [4, 1, 2, 5], 4),
                  ([7, 0, 8, 8], 1, None, -1, [0, 6, 7], 1)]
        for seq, (ids, cur, pred, nxt, want, copies) in enumerate(layers, start=2):
            dev_ids = torch.tensor(ids, dtype=torch.int32, device="cuda")
            dev_pred = torch.tensor(pred or [0], dtype=torch.int32, device="cuda")
            lib.call("ps_fetcher_submit_spec", f, seq, host, nbytes, nbytes, slots.data_ptr(), nbytes, n_slots,
                     host, nbytes, nbytes)
            lib.call("ps_moe_publish_spec", f, dev_ids.data_ptr(), k, E, slotmap.data_ptr(), seq,
                     dev_pred.data_ptr(), S, state.data_ptr(), cur, nxt, k, sor.data_ptr(), stream())
            lib.call("ps_wait_flag", f, seq, stream())
            torch.cuda.synchronize()
            routed = sorted(set(ids))
            got_sor = sor.cpu().numpy()[:len(routed)].tolist()
            assert got_sor == want, (seq, got_sor, want)
            got = slots.cpu().numpy().reshape(n_slots, nbytes)
            for r, e in enumerate(routed):
                assert np.array_equal(got[got_sor[r]], src[e]), (seq, r, e)
            m = slotmap.cpu().numpy()
            for e in range(E):
                assert m[e] == (routed.index(e) if e in routed else -1)
            b = ctypes.c_longlong()
            lib.call("ps_fetcher_seq_bytes", f, seq, ctypes.byref(b))
            assert b.value == copies * nbytes, (seq, b.value)
        n, b, err = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int()
        lib.call("ps_fetcher_info", f, None, None, ctypes.byref(n), ctypes.byref(b), ctypes.byref(err))
        assert (n.value, err.value) == (11, 0)
        lib.host_free(host)
    finally:
        lib.call("ps_fetcher_destroy", f)


@pytest.mark.parametrize("N,K,t,epi", [(512, 4096, 1, 0), (1000, 2048, 2, 1), (640, 14336, 1, 0),
                                       (256, 4096, 8, 2), (300, 512, 4, 0), (4096, 768, 1, 1)])
def test_gemv_coded_bit_identical(N, K, t, epi):
    """ps_gemv_bf16c on exponent-coded weights (runtime/wcomp.py, 12 bits/weight, per-row
    base exponent, escapes in each row's trailer) is bit-identical to ps_gemv_bf16 on the
    bf16 weights: zeros, denormals, huge and tiny values outside a row's 15-exponent
    window, a row scaled by 2^20 (its own base) and a row with 40 escapes."""
    from paper_2604_26334_b200.runtime import wcomp
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(N + K)
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * 0.03
    W[0, :7] = 0.0
    W[1, 3] = 1e-30
    W[2, 11] = 3.0e4
    W[3] *= 2.0 ** 20
    W[4, 5:45] = 1e-12
    W[N - 1, K - 1] = -1e-38
    bits = W.view(torch.int16).cpu().numpy().view(np.uint16)
    coded, tb = wcomp.encode(bits)
    assert tb >= 16 * 11                         # 40 escapes + header
    assert np.array_equal(wcomp.decode(coded, K), bits)
    Wc = torch.from_numpy(coded).cuda()
    x = torch.randn(t, K, device="cuda", generator=g)
    rows = N // 2 if epi == 2 else N
    y0 = torch.randn(t, rows, device="cuda", generator=g)
    ya, yb = y0.clone(), y0.clone()
    s = stream()
    lib.call("ps_gemv_bf16_cfg", x.data_ptr(), K, t, W.data_ptr(), N, K, K, ya.data_ptr(), rows, epi, s, -1, 0, 0)
    lib.call("ps_gemv_bf16c", x.data_ptr(), K, t, Wc.data_ptr(), N, K, coded.shape[1], yb.data_ptr(), rows, epi, s)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)


@pytest.mark.parametrize("N,K,t,epi", [(6144, 4096, 32, 0), (4096, 14336, 32, 1), (28672, 4096, 16, 2),
                                       (1000, 2048, 9, 0), (300, 512, 32, 1), (128256, 4096, 32, 0),
                                       (4096, 768, 24, 2)])
def test_gemv_tc_one_pass_fp32_faithful(N, K, t, epi):
    """Decode batches of 9..32 tokens on tcgen05 (ps_gemv_tc): W read once, x split into
    three bf16 planes -> fp32-faithful (within 1e-5 of an fp64 reference, like the fp32
    CUDA-core GEMV); the exponent-coded variant is bit-identical to the bf16 one, escapes
    and per-row bases included; split-K shapes (N / 128 < SMs) and partial row tiles."""
    from paper_2604_26334_b200.runtime import wcomp
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(N + K + t)
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * 0.03
    W[0, :7] = 0.0
    W[3] *= 2.0 ** 20
    W[N - 1, K - 1] = -1e-38
    x = torch.randn(t, K, device="cuda", generator=g)
    rows = N // 2 if epi == 2 else N
    y0 = torch.randn(t, rows, device="cuda", generator=g)
    ws_n = C.c_longlong()
    lib.call("ps_gemv_tc_workspace", N, K, C.byref(ws_n))
    ws = torch.empty(ws_n.value, dtype=torch.uint8, device="cuda")
    ya, yb, yc = y0.clone(), y0.clone(), y0.clone()
    s = stream()
    lib.call("ps_gemv_tc", x.data_ptr(), K, t, W.data_ptr(), N, K, K, 0, ya.data_ptr(), rows, epi,
             ws.data_ptr(), ws.numel(), s)
    bits = W.view(torch.int16).cpu().numpy().view(np.uint16)
    coded, tb = wcomp.encode(bits)
    Wc = torch.from_numpy(coded).cuda()
    lib.call("ps_gemv_tc", x.data_ptr(), K, t, Wc.data_ptr(), N, K, coded.shape[1], 1, yb.data_ptr(), rows, epi,
             ws.data_ptr(), ws.numel(), s)
    lib.call("ps_gemv_bf16", x.data_ptr(), K, t, W.data_ptr(), N, K, K, yc.data_ptr(), rows, epi, s)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)                      # coded == bf16, bit for bit
    full = x.double() @ W.double().T                # [t, N]
    if epi == 2:
        ref = torch.nn.functional.silu(full[:, 0::2]) * full[:, 1::2]
    elif epi == 1:
        ref = y0.double() + full
    else:
        ref = full
    scale = ref.abs().max()
    assert float((ya.double() - ref).abs().max() / scale) < 1e-5
    assert float((yc.double() - ref).abs().max() / scale) < 1e-5


@pytest.mark.parametrize("E,k,d,eff", [(32, 8, 2048, 768), (16, 4, 512, 256)])
def test_moe_decode_experts_coded_bit_identical(E, k, d, eff):
    """ps_moe_decode_experts_c on exponent-coded experts (every expert of the group one
    row size: the group's largest trailer) equals ps_moe_decode_experts on the bf16
    experts bit for bit, escapes included, through a fetcher-style slot map."""
    from paper_2604_26334_b200.runtime import wcomp
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(E * 7 + d)
    x = torch.randn(1, d, device="cuda", generator=g)
    Wgu = (torch.randn(E, 2 * eff, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
    Wd = (torch.randn(E, d, eff, device="cuda", generator=g) / eff ** 0.5).to(torch.bfloat16)
    Wgu[1, 3, :5] = 0.0
    Wd[2, 7] *= 2.0 ** 24
    bits_gu = [Wgu[e].view(torch.int16).cpu().numpy().view(np.uint16) for e in range(E)]
    bits_d = [Wd[e].view(torch.int16).cpu().numpy().view(np.uint16) for e in range(E)]
    tg = max(wcomp._trailer_or_none(b) for b in bits_gu)
    td = max(wcomp._trailer_or_none(b) for b in bits_d)
    up = lambda n: (n + 255) // 256 * 256  # noqa: E731
    gu_rb, d_rb = wcomp.row_bytes(d, tg), wcomp.row_bytes(eff, td)
    down_off = up(2 * eff * gu_rb)
    cstride = up(down_off + d * d_rb)
    cblob = np.zeros(E * cstride, np.uint8)
    for e in range(E):
        wcomp.encode(bits_gu[e], out=cblob[e * cstride:], trailer=tg)
        wcomp.encode(bits_d[e], out=cblob[e * cstride + down_off:], trailer=td)
    blob = torch.cat([torch.cat([Wgu[e].reshape(-1), Wd[e].reshape(-1)]) for e in range(E)]).contiguous()
    stride = (2 * eff * d + d * eff) * 2
    ids = torch.tensor(np.random.default_rng(E).choice(E, k, replace=False).astype(np.int32), device="cuda")
    ids[0] = 1
    ids[1] = 2 if k > 1 else ids[1]
    w = torch.rand(k, device="cuda", generator=g)
    sb = up(stride)
    slots = torch.zeros(k * sb, dtype=torch.uint8, device="cuda")
    cslots = torch.zeros(k * sb, dtype=torch.uint8, device="cuda")
    smap = torch.full((E,), -1, dtype=torch.int32, device="cuda")
    cb = torch.from_numpy(cblob).cuda()
    bb = blob.view(torch.uint8)
    for j, e in enumerate(ids.tolist()):
        sl = k - 1 - j
        slots[sl * sb:sl * sb + stride] = bb[e * stride:(e + 1) * stride]
        cslots[sl * sb:sl * sb + cstride] = cb[e * cstride:(e + 1) * cstride]
        smap[e] = sl
    h = torch.zeros(k, eff, device="cuda")
    y0 = torch.randn(1, d, device="cuda", generator=g)
    ya, yb = y0.clone(), y0.clone()
    s = stream()
    lib.call("ps_moe_decode_experts", x.data_ptr(), ids.data_ptr(), k, smap.data_ptr(), slots.data_ptr(), sb, 0,
             2 * eff * d * 2, eff, d, h.data_ptr(), w.data_ptr(), ya.data_ptr(), s)
    lib.call("ps_moe_decode_experts_c", x.data_ptr(), ids.data_ptr(), k, smap.data_ptr(), cslots.data_ptr(), sb, 0,
             down_off, eff, d, gu_rb, d_rb, h.data_ptr(), w.data_ptr(), yb.data_ptr(), s)
    torch.cuda.synchronize()
    assert torch.equal(ya, yb)


@pytest.mark.parametrize("N,K", [(300, 4096), (64, 14336), (1000, 256), (5, 2048)])
def test_gpu_encoder_byte_identical(N, K):
    """ps_wencode_stats + ps_wencode_rows (csrc/wencode.cu) produce exactly the bytes of
    wcomp.encode (the numpy reference): per-row bases, the best-covering window of a row
    with an outlier (recheck path), escapes in ascending column order, 0xFF padding, and
    the same escape counts; also through GpuEncoder's chunked H2D / D2H path."""
    from paper_2604_26334_b200.runtime import wcomp
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(N * 7 + K)
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * 0.03
    W[0, :7] = 0.0
    W[1, 3] = 1e-30
    W[2, 11] = 3.0e4                      # one outlier far above the bulk: recheck picks the bulk's window
    W[3] *= 2.0 ** 20
    W[4, 5:45] = 1e-12                    # 40 escapes below the window
    W[N - 1, K - 1] = -1e-38
    W[min(N - 1, 5), :20] *= 2.0 ** -30   # 20 weights far below the window
    bits = W.view(torch.int16).cpu().numpy().view(np.uint16)
    want = wcomp.encode(bits, max_escapes=1 << 20)
    assert want is not None
    coded, tb = want
    base = torch.empty(N, dtype=torch.int32, device="cuda")
    count = torch.empty(N, dtype=torch.int32, device="cuda")
    s = stream()
    lib.call("ps_wencode_stats", W.data_ptr(), N, K, K, base.data_ptr(), count.data_ptr(), s)
    torch.cuda.synchronize()
    exp = ((bits >> 7) & 0xFF).astype(np.uint8)
    assert np.array_equal(base.cpu().numpy(), wcomp.row_bases(exp).astype(np.int32))
    top = int(count.max().item())
    assert wcomp.trailer_bytes(top) == tb
    out = torch.full((N, coded.shape[1]), 0x5A, dtype=torch.uint8, device="cuda")
    lib.call("ps_wencode_rows", W.data_ptr(), N, K, K, base.data_ptr(), tb, out.data_ptr(), coded.shape[1], s)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy(), coded)
    if top <= wcomp.MAX_ESCAPES:   # GpuEncoder: chunked through pinned host memory
        host_src = lib.host_alloc(bits.nbytes, mapped=False)
        host_dst = lib.host_alloc(coded.nbytes, mapped=False)
        try:
            C.memmove(host_src, bits.ctypes.data, bits.nbytes)
            enc = wcomp.GpuEncoder(chunk_bytes=max(2 * K, (N // 3) * 2 * K))
            assert enc.max_escapes(host_src, N, K) == top
            enc.encode_to(host_src, N, K, tb, host_dst)
            enc.close()
            got = np.ctypeslib.as_array((C.c_uint8 * coded.nbytes).from_address(host_dst)).reshape(coded.shape)
            assert np.array_equal(got, coded)
        finally:
            lib.host_free(host_src)
            lib.host_free(host_dst)


@pytest.mark.parametrize("N,K", [(130, 768), (70, 512), (1, 256), (65, 1024)])
def test_hx_encoder_and_expand_exact(N, K):
    """Huffman-coded exponents (csrc/hx.cu): the GPU encoder (ps_hx_stats / sizes / write)
    writes exactly the bytes of the CPU reference (runtime/hxcodec.encode), and
    ps_hx_expand restores the bf16 bits exactly — whole matrix and a run of blocks
    starting mid-matrix — zeros, denormals, an outlier row and 2^20-scaled rows included."""
    from paper_2604_26334_b200.runtime import hxcodec as hx
    lib = L()
    g = torch.Generator(device="cuda").manual_seed(N * 13 + K)
    W = (torch.rand(N, K, device="cuda", generator=g) * 2 - 1).to(torch.bfloat16) * 0.03
    W[0, :7] = 0.0
    if N > 3:
        W[1, 3] = 1e-30
        W[2, 11] = 3.0e4
        W[3] *= 2.0 ** 20
    bits = W.view(torch.int16).cpu().numpy().view(np.uint16)
    blob, offs, table = hx.encode(bits)
    enc = hx.GpuHxEncoder()
    fill = lambda dst, r0, r1: lib.memcpy_async(dst, W.data_ptr() + r0 * K * 2, (r1 - r0) * K * 2,  # noqa: E731
                                                stream())
    m = enc.plan(fill, N, K)
    assert np.array_equal(m.table, table) and np.array_equal(m.block_off, offs)
    host = lib.host_alloc(m.nbytes, mapped=False)
    try:
        enc.write(fill, m, host)
        got = np.ctypeslib.as_array((C.c_uint8 * m.nbytes).from_address(host)).copy()
    finally:
        lib.host_free(host)
    assert np.array_equal(got, blob)
    dev = torch.from_numpy(blob).cuda()
    lut = torch.from_numpy(m.lut.view(np.int32)).cuda()
    for b0 in (0, 1):
        if b0 * hx.BLOCK_ROWS >= N:
            continue
        nb = len(offs) - 1 - b0
        rel = torch.from_numpy((offs[b0:-1] - offs[b0]).astype(np.uint32).view(np.int32)).cuda()
        rows = N - b0 * hx.BLOCK_ROWS
        out = torch.full((rows, K), -1, dtype=torch.int16, device="cuda")
        lib.call("ps_hx_expand", dev.data_ptr() + int(offs[b0]), rel.data_ptr(), rows, K, lut.data_ptr(),
                 out.data_ptr(), K, stream())
        torch.cuda.synchronize()
        assert nb >= 1
        assert np.array_equal(out.cpu().numpy().view(np.uint16), bits[b0 * hx.BLOCK_ROWS:]), b0
