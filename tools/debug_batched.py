import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.planning.graph import total_model_bytes
from paper_2604_26334_b200.runtime import executor as X, lib as L
from paper_2604_26334_b200.runtime.engine import Engine
orig = X.Executor.run_pass
def traced(self, ps):
    r = orig(self, ps)
    self.synchronize()
    x = self.arena.tensor(self.x, ps.T * self.d * 4).view(torch.float32)
    R = len(ps.sample)
    lg = self.arena.tensor(self.logits, max(R, 1) * self.V * 4).view(torch.float32)
    kinds = {m for m, _ in self.residency.values()}
    print("PASS tier", self.tier, "slots", ps.slots, "n_new", ps.n_new, "p0", ps.p0, "sample", ps.sample,
          "x_nan", bool(torch.isnan(x).any()), "logit_nan", bool(torch.isnan(lg).any()), "modes", kinds,
          "kv", sorted(set(self.kv_mode.values())), flush=True)
    return r
X.Executor.run_pass = traced
tiny = catalog.builtin_model("tiny-llama")
prompts = [np.random.default_rng(30 + i).integers(0, tiny.vocab_size, n).astype(np.int32) for i, n in enumerate([100, 60, 128])]
eng = Engine(tiny, budget_bytes=0.5 * total_model_bytes(tiny), context_len=160, batch=3)
print({t: p.kind.value for t, p in eng.plans.items()})
res = eng.generate(prompts, gen_len=8)
print(res.tokens)
