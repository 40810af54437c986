"""Device timeline of steady-state decode passes from CUPTI (torch.profiler): every
kernel and memcpy of the process — including libpshard's, launched through ctypes,
and the fetcher thread's copies — with GPU start/end times (nsys is not installed).

    python tools/cupti_trace.py --config 3 --passes 1 --out gpurun_out/cupti_cfg3.json
Prints per-kernel-name totals and the idle gaps of the compute stream."""
import argparse
import collections
import json
import os
import sys

import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_26334_b200.runtime.engine import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--passes", type=int, default=1)
ap.add_argument("--skip", type=int, default=3)
ap.add_argument("--out", default="gpurun_out/cupti.json")
a = ap.parse_args()
model, budget, prompt, gen, batch, desc = bench.CONFIGS[a.config]
if budget is None:   # config 1: 50 % of the plan's weight bytes (bench.py)
    from paper_2604_26334_b200.planning import catalog
    from paper_2604_26334_b200.planning.graph import total_model_bytes
    budget = 0.5 * total_model_bytes(catalog.builtin_model(model))
eng = Engine(model, budget_bytes=budget, context_len=prompt + gen, batch=batch)
prompts = [np.random.default_rng(i).integers(0, eng.spec.vocab_size, prompt).astype(np.int32)
           for i in range(batch)]
eng.prepare([prompt] * batch, a.skip + a.passes + 1)
prof = profile(activities=[ProfilerActivity.CUDA])
state = {}


def on_pass(i, tier, ex):
    if i == a.skip:
        ex.synchronize()
        prof.__enter__()
        state["on"] = True
    elif i == a.skip + a.passes and state.get("on"):
        ex.synchronize()
        prof.__exit__(None, None, None)
        state["on"] = False


res = eng.generate(prompts, gen_len=a.skip + a.passes + 1, on_pass=on_pass)
if state.get("on"):
    eng.executor.synchronize()
    prof.__exit__(None, None, None)
prof.export_chrome_trace(a.out)
ev = [e for e in json.load(open(a.out))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy")]
by = collections.defaultdict(lambda: [0, 0.0])
for e in ev:
    k = e["name"].split("(")[0][:60]
    by[k][0] += 1
    by[k][1] += e["dur"]
top = sorted(by.items(), key=lambda kv: -kv[1][1])[:25]
streams = collections.defaultdict(list)
for e in ev:
    streams[(e.get("args", {}).get("stream"), e["cat"])].append((e["ts"], e["ts"] + e["dur"]))
summary = {"config": desc, "passes": a.passes,
           "pass_ms": [round(p[2] * 1e3, 2) for p in res.passes[a.skip:a.skip + a.passes]],
           "top": [{"name": k, "n": n, "total_us": round(t, 1), "avg_us": round(t / n, 2)} for k, (n, t) in top],
           "streams": {}}
for key, iv in streams.items():
    iv.sort()
    busy = sum(b - a_ for a_, b in iv)
    span = iv[-1][1] - iv[0][0]
    gaps = [iv[i + 1][0] - iv[i][1] for i in range(len(iv) - 1)]
    summary["streams"][f"{key[0]}:{key[1]}"] = {"ops": len(iv), "busy_us": round(busy, 1), "span_us": round(span, 1),
                                                "gap_total_us": round(sum(g for g in gaps if g > 0), 1)}
print(json.dumps(summary, indent=1))
eng.close()
