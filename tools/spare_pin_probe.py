"""Arena accounting of a BASELINE config's decode tier: capacity, pinned + spare-pinned
bytes, activations, ring and what is left (GPU: builds the executor)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2604_26334_b200.runtime.engine import Engine  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
model, budget, prompt, gen, batch, desc = bench.CONFIGS[cfg]
eng = Engine(model, budget_bytes=budget, context_len=prompt + gen, batch=batch)
eng.prepare([prompt] * batch, gen)
ex = eng.executor
a = ex.arena
spare = sum(ex._phys_bytes(ex.shards[s]) for s in ex.spare_pinned)
print({"capacity_MB": a.capacity >> 20, "low_MB": a.low >> 20, "high_used_MB": (a.capacity - a.high) >> 20,
       "free_MB": a.free_bytes >> 20, "ring_MB": (ex.ring.capacity >> 20) if ex.ring else 0,
       "chunk_MB": ex.chunk >> 20, "ring_keep_pieces": ex.ring_keep_pieces, "spare_MB": spare >> 20,
       "spare": [(ex.shards[s].kind.name, ex.shards[s].layer_index) for s in ex.spare_pinned],
       "high_marks": {k: (v[1] >> 20) for k, v in a.high_marks.items()}})
eng.close()
