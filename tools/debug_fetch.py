import sys, os, tempfile
sys.path.insert(0, ".")
import numpy as np
from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.planning.graph import total_model_bytes
from paper_2604_26334_b200.runtime.engine import Engine

def run(model, frac, ckpt_dir=None, export=None):
    spec = catalog.builtin_model(model)
    budget = frac * total_model_bytes(spec)
    prompt = np.random.default_rng(5).integers(0, spec.vocab_size, 40).astype(np.int32)
    if ckpt_dir:
        eng = Engine(None, budget_bytes=budget, context_len=160, checkpoint=ckpt_dir)
    else:
        eng = Engine(spec, budget_bytes=budget, context_len=160)
    try:
        res = eng.generate([prompt], gen_len=8)
        print(model, frac, "ckpt" if ckpt_dir else "rand", "tokens", res.tokens[0], "fetch", eng.executor.fetcher_stats(), flush=True)
        if export:
            eng.weights.export(export)
    except Exception as e:
        print("FAILED", model, frac, "ckpt" if ckpt_dir else "rand", repr(e)[:300], "fetch", eng.executor.fetcher_stats() if eng.executor else None, flush=True)
        raise
    finally:
        pass
    eng.close()

order = sys.argv[1]
d1, d2 = tempfile.mkdtemp(), tempfile.mkdtemp()
if order == "a":
    run("tiny-llama", 0.6, export=d1); run("tiny-llama", 0.6, ckpt_dir=d1)
run("tiny-moe", 1.0, export=d2)
run("tiny-moe", 1.0, ckpt_dir=d2)
