import os, sys
sys.path.insert(0, ".")
import numpy as np
from paper_2604_26334_b200.runtime.engine import Engine
eng = Engine("llama3.1-8b", budget_bytes=4e9, context_len=2304)
eng.prepare([2048], 8)
ex = eng.executor
print("keep", ex.ring_keep_pieces, "capacity", ex.arena.capacity, "persist_high", ex.persist_high, "free_now", ex.arena.free_bytes,
      "ring", ex.ring.capacity if ex.ring else None, "spare_pinned", len(ex.spare_pinned),
      [ (ex.shards[s].kind.name, ex.shards[s].layer_index) for s in ex.spare_pinned][:8], flush=True)
eng.close()
