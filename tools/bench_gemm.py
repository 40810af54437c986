"""Time the tcgen05 GEMM variants (1-CTA tile kernel vs persistent CTA-pair
kernel) and torch.matmul (cuBLAS) on the prefill shapes the executor launches.

CUDA events on the launching stream, L2 flushed (256 MB write) before each
timed launch, best and mean of `reps`. Prints one JSON line per shape/variant:
achieved TFLOP/s and the fraction of MEASURED_PEAKS.json's burst bf16 peak."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.runtime import lib as L

PEAK = json.load(open("MEASURED_PEAKS.json"))["bf16_tflops"] if os.path.exists("MEASURED_PEAKS.json") else 1590.0
# (M, N, K, epilogue, what): L8 prefill 2048 tokens (config 2) and 16384 tokens (config 4)
SHAPES = [(2048, 6144, 4096, 0, "L8 wqkv t=2048"), (2048, 4096, 4096, 1, "L8 wo t=2048"),
          (2048, 28672, 4096, 2, "L8 wgu t=2048"), (2048, 4096, 14336, 1, "L8 wdown t=2048"),
          (16384, 6144, 4096, 0, "L8 wqkv t=16384"), (16384, 28672, 4096, 2, "L8 wgu t=16384"),
          (16384, 4096, 14336, 1, "L8 wdown t=16384"), (8192, 8192, 8192, 3, "8192^3 bf16-out")]


def run(M, N, K, epi, variant, reps=10):
    A = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    B = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
    if epi == 2:
        C = torch.zeros(M, N // 2, device="cuda", dtype=torch.bfloat16); ldc = N // 2
    elif epi == 3:
        C = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16); ldc = N
    else:
        C = torch.zeros(M, N, device="cuda"); ldc = N
    flush = torch.ones(64 << 20, dtype=torch.float32, device="cuda")  # 256 MB > L2
    s = torch.cuda.current_stream().cuda_stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for i in range(reps + 3):
        flush.sum()
        e0.record()
        if variant == "cublas":
            torch.matmul(A, B.T)
        else:
            L.call("ps_gemm_bf16_cfg", A.data_ptr(), M, K, K, B.data_ptr(), N, K, C.data_ptr(), ldc, epi, s,
                   variant)
        e1.record()
        torch.cuda.synchronize()
        if i >= 3:
            ts.append(e0.elapsed_time(e1) / 1e3)
    err = None
    if variant != "cublas" and epi in (0, 3):
        ref = A[:512].float() @ B.float().T
        err = float((C[:512].float() - ref).abs().max() / ref.abs().max())
    fl = 2.0 * M * N * K
    return fl / min(ts) / 1e12, fl / (sum(ts) / len(ts)) / 1e12, min(ts) * 1e6, err


for M, N, K, epi, what in SHAPES:
    for v in (1, 2, "cublas"):
        best, mean, us, err = run(M, N, K, epi, v)
        print(json.dumps({"shape": what, "M": M, "N": N, "K": K, "epi": epi, "variant": v,
                          "tflops_best": round(best, 1), "tflops_mean": round(mean, 1),
                          "frac_of_measured_peak": round(best / PEAK, 3), "us": round(us, 1),
                          "rel_err": err}), flush=True)
