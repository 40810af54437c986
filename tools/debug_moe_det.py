"""Determinism probe of the tiny-moe (expert width 256) decode: the same generate run
repeated under switch combinations; prints the greedy ids of each run."""
import dataclasses
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.planning import catalog  # noqa: E402
from paper_2604_26334_b200.planning.graph import MoeSpec, total_model_bytes  # noqa: E402
from paper_2604_26334_b200.runtime.engine import Engine  # noqa: E402

base = catalog.builtin_model("tiny-moe")
spec = dataclasses.replace(base, moe=MoeSpec(base.moe.n_experts, base.moe.top_k, 256))
prompt = np.random.default_rng(17).integers(0, spec.vocab_size, 24).astype(np.int32)
combos = [dict(), dict(PS_CODED_EXPERTS="0"), dict(PS_CODED_RESIDENT="0"), dict(PS_CODED="0"),
          dict(PS_GAPFILL="0"), dict(PS_MOE_DECODE="0"), dict(PS_CODED_EXPERTS="0", PS_CODED_RESIDENT="0")]
for combo in combos:
    for rep in range(2):
        for k in ("PS_CODED_EXPERTS", "PS_CODED_RESIDENT", "PS_CODED", "PS_GAPFILL", "PS_MOE_DECODE"):
            os.environ.pop(k, None)
        os.environ.update(combo)
        eng = Engine(spec, budget_bytes=1.0 * total_model_bytes(spec), context_len=160)
        res = eng.generate([prompt], gen_len=12)
        lg = eng.logits()[0]
        print(combo, rep, res.tokens[0].tolist(), res.row_modes[0][-12:], float(np.abs(lg).sum()), flush=True)
        eng.close()
