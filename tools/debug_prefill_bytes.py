"""Which shards a prefill pass streams, and in which form (debug aid): tiny-llama at a
small budget, PS_HX=0, PS_CODED_PREFILL 0 vs 1."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.planning import catalog  # noqa: E402
from paper_2604_26334_b200.planning.graph import total_model_bytes  # noqa: E402
from paper_2604_26334_b200.runtime.engine import Engine  # noqa: E402

spec = catalog.builtin_model("tiny-llama")
prompt = np.random.default_rng(33).integers(0, spec.vocab_size, 128).astype(np.int32)
os.environ["PS_HX"] = "0"
os.environ["PS_CODED_RESIDENT"] = "0"
for frac in (0.25, 0.5):
    for cp in ("0", "1"):
        os.environ["PS_CODED_PREFILL"] = cp
        eng = Engine(spec, budget_bytes=frac * total_model_bytes(spec), context_len=160, chunk_bytes=1 << 20)
        eng._ensure_executor(160)
        ex = eng.executor
        log = []
        orig_shard = ex._shard

        def shard(sid, consumers, T, _o=orig_shard, _ex=ex, _log=log):
            if T > 32:
                mode = _ex.residency[sid][0]
                coded = _ex.coded is not None and sid in _ex.coded.tensors
                _log.append((sid, mode, coded, bool(_ex.expand), _ex._coded_prefill()))
            return _o(sid, consumers, T)
        ex._shard = shard
        res = eng.generate([prompt], gen_len=4)
        pre = [s for s in ex.stats if s.T > 32]
        print(frac, cp, "streamed", sum(s.bytes_streamed for s in pre), "kv", sum(s.kv_bytes for s in pre),
              "zc", sum(s.zero_copy_bytes for s in pre), "form", getattr(ex, "resident_form", None))
        print("   ", log)
        eng.close()
