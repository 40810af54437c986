"""Copy/compute overlap timeline of steady-state decode passes (Chrome trace).

    python tools/trace_decode.py --config 2 --passes 2 --out gpurun_out/trace_cfg2.json

Attaches a Tracer after the prompt pass and the first decode passes, records
--passes decode passes, writes the Chrome trace and prints the overlap summary."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402  (config table)
from paper_2604_26334_b200.runtime.engine import Engine  # noqa: E402
from paper_2604_26334_b200.runtime.tracer import Tracer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--passes", type=int, default=2)
ap.add_argument("--skip", type=int, default=3, help="passes (incl. the prompt pass) before tracing")
ap.add_argument("--out", default="gpurun_out/trace.json")
a = ap.parse_args()
model, budget, prompt, gen, batch, desc = bench.CONFIGS[a.config]
eng = Engine(model, budget_bytes=budget, context_len=prompt + gen, batch=batch)
prompts = [np.random.default_rng(i).integers(0, eng.spec.vocab_size, prompt).astype(np.int32)
           for i in range(batch)]
n_gen = a.skip + a.passes + 1
eng.prepare([prompt] * batch, n_gen)
tracer = Tracer()


def on_pass(i, tier, ex):
    if i == a.skip:
        ex.attach_tracer(tracer)
    elif i == a.skip + a.passes:
        ex.attach_tracer(None)


res = eng.generate(prompts, gen_len=n_gen, on_pass=on_pass)
summary = tracer.dump(a.out)
summary.update({"config": desc, "traced_passes": a.passes,
                "pass_ms": [round(p[2] * 1e3, 2) for p in res.passes[a.skip:a.skip + a.passes]]})
print(json.dumps(summary))
tracer.close()
eng.close()
