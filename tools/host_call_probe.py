"""Where does the host spend a decode pass's enqueue time? Wraps lib.call and sums
wall time per C-ABI entry point over steady-state passes (config 3 by default)."""
import collections, json, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
from paper_2604_26334_b200.runtime import lib as L
from paper_2604_26334_b200.runtime.engine import Engine
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
model, budget, prompt, gen, batch, desc = bench.CONFIGS[cfg]
eng = Engine(model, budget_bytes=budget, context_len=prompt + gen, batch=batch)
prompts = [np.random.default_rng(i).integers(0, eng.spec.vocab_size, prompt).astype(np.int32) for i in range(batch)]
eng.prepare([prompt] * batch, 8)
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
orig = L.call
state = {"on": False}
def timed(name, *args):
    if not state["on"]:
        return orig(name, *args)
    t0 = time.perf_counter()
    r = orig(name, *args)
    dt = time.perf_counter() - t0
    e = tot[name]; e[0] += 1; e[1] += dt; e[2] = max(e[2], dt)
    return r
L.call = timed
def on_pass(i, tier, ex):
    state["on"] = i >= 4
res = eng.generate(prompts, gen_len=8, on_pass=on_pass)
print(json.dumps({k: {"n": v[0], "ms": round(v[1] * 1e3, 2), "max_ms": round(v[2] * 1e3, 3)}
                  for k, v in sorted(tot.items(), key=lambda kv: -kv[1][1])}, indent=0))
eng.close()
