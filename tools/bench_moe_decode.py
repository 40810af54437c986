"""Warm per-kernel times of the one-token MoE decode path at the Qwen3-30B-A3B shape
(E=128, k=8, d=2048, eff=768; 1.2 GB of experts in VRAM, routed sets rotated so
no call reads its experts from L2), against the general plan/gu/down/combine path.

    python tools/bench_moe_decode.py [--iters 50]"""
import argparse
import collections
import json
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.runtime import lib as L  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=50)
ap.add_argument("--d", type=int, default=2048)
ap.add_argument("--eff", type=int, default=768)
ap.add_argument("--k", type=int, default=8)
a = ap.parse_args()
E, k, d, eff = 128, a.k, a.d, a.eff
lib = L
stride = 3 * d * eff * 2
blob = torch.randn(E * stride // 2, device="cuda").to(torch.bfloat16) * 0.02
x = torch.randn(d, device="cuda")
y = torch.zeros(d, device="cuda")
h = torch.zeros(k, eff, device="cuda")
out = torch.zeros(k, d, device="cuda")
w = torch.full((k,), 1.0 / k, device="cuda")
sets = [torch.arange(i * k, (i + 1) * k, dtype=torch.int32, device="cuda") for i in range(E // k)]
n = __import__("ctypes").c_longlong()
lib.call("ps_moe_plan_ints", k, E, __import__("ctypes").byref(n))
plan = torch.zeros(n.value, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream


def fused(ids):
    lib.call("ps_moe_decode_experts", x.data_ptr(), ids.data_ptr(), k, None, blob.data_ptr(), stride, 0,
             2 * eff * d * 2, eff, d, h.data_ptr(), w.data_ptr(), y.data_ptr(), s)


def general(ids):
    lib.call("ps_moe_plan", ids.data_ptr(), k, E, plan.data_ptr(), s)
    lib.call("ps_moe_expert_gu", x.data_ptr(), d, 0, plan.data_ptr(), E, k, k, blob.data_ptr(), stride, 0,
             eff, d, h.data_ptr(), 0, E, s)
    lib.call("ps_moe_expert_down", h.data_ptr(), plan.data_ptr(), E, k, blob.data_ptr(), stride, 2 * eff * d * 2,
             eff, d, out.data_ptr(), 0, E, s)
    lib.call("ps_moe_combine", out.data_ptr(), plan.data_ptr(), E, k, w.data_ptr(), 1, k, d, y.data_ptr(), d, s)


res = {"chunk": os.environ.get("PS_MD_CHUNK", "default"), "d": d, "eff": eff, "k": k}
for name, fn in (("fused", fused),) + ((("general", general),) if os.environ.get("GENERAL", "1") == "1" else ()):
    for i in range(10):
        fn(sets[i % len(sets)])
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for i in range(a.iters):
            fn(sets[i % len(sets)])
        torch.cuda.synchronize()
    by = collections.defaultdict(list)
    for e in prof.events():
        if e.device_type.name == "CUDA":
            by[e.name.split("(")[0].split("<")[0]].append(e.device_time_total if hasattr(e, "device_time_total")
                                                          else e.cuda_time_total)
    res[name] = {k_: round(sum(v) / len(v), 2) for k_, v in by.items()}
    res[name]["sum_us"] = round(sum(res[name].values()), 2)
res["bytes_per_call"] = k * stride
res["fused_TBps"] = round(k * stride / res["fused"]["sum_us"] / 1e6, 2)
print(json.dumps(res, indent=1))
