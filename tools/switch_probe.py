"""Print each tier's resident set (plan pins + spare pins) and the relocation plan of
the decode <-> prefill switches for a BASELINE config (GPU: builds the executor)."""
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2604_26334_b200.runtime.engine import Engine  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
model, budget, prompt, gen, batch, desc = bench.CONFIGS[cfg]
eng = Engine(model, budget_bytes=budget, context_len=prompt + gen, batch=batch)
eng.prepare([prompt] * batch, gen)
ex, mm = eng.executor, eng.migration
dec, pre = eng.pick_tier(batch), eng.pick_tier(prompt * batch)
for t in (dec, pre):
    pins = ex.pins_for(t)
    plan_p = {p.shard_id for p in eng.plans[t].placements if p.residency.name == "VRAM_PINNED"}
    desc = [(ex.shards[s].kind.name[:4], ex.shards[s].layer_index, "P" if s in plan_p else "S") for s in pins]
    print(t, len(pins), desc)
for a, b in ((dec, pre), (pre, dec)):
    print(a, "->", b, "h2d/d2h/d2d GB", [round(x / 1e9, 3) for x in mm.moves(a, b, prompt)])
eng.close()
