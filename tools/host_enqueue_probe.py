"""Host enqueue time of each pass (time inside Executor.run_pass) beside its device time:
if they are close, the pass is host-bound (the GPU waits for the Python host)."""
import json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2604_26334_b200.runtime.engine import Engine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
model, budget, prompt, gen, batch, desc = bench.CONFIGS[cfg]
eng = Engine(model, budget_bytes=budget, context_len=prompt + gen, batch=batch)
prompts = [np.random.default_rng(i).integers(0, eng.spec.vocab_size, prompt).astype(np.int32) for i in range(batch)]
eng.prepare([prompt] * batch, 8)
host_ms = []
def on_pass(i, tier, ex):
    if not hasattr(ex, "_orig_run_pass"):
        ex._orig_run_pass = ex.run_pass
        def timed(ps):
            t0 = time.perf_counter()
            r = ex._orig_run_pass(ps)
            host_ms.append((time.perf_counter() - t0) * 1e3)
            return r
        ex.run_pass = timed
res = eng.generate(prompts, gen_len=8, on_pass=on_pass)
print(json.dumps({"config": cfg, "host_enqueue_ms": [round(h, 2) for h in host_ms],
                  "device_ms": [round(p[2] * 1e3, 2) for p in res.passes]}))
eng.close()
