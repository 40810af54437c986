"""Planner estimates (synthetic vs measured B200 profile) beside the measured
decode step and prefill pass of each BASELINE config (profiles/r01_bench_cfg*.json)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_26334_b200.planning import catalog
from paper_2604_26334_b200.planning.costdb import load_profile, synth_profile
from paper_2604_26334_b200.planning.graph import total_model_bytes
from paper_2604_26334_b200.planning.placement import reachable_tiers

m = catalog.builtin_machine("b200")
dbs = {"plan_synthetic_profile": synth_profile(m), "plan_b200_measured_profile": load_profile("profiles/r01_b200_measured.profile")}
CFG = [(1, "tiny-llama", None, 128, 32, 1, "r01_bench_cfg1_tiny.json"),
       (2, "llama3.1-8b", 4e9, 2048, 256, 1, "r01_bench_cfg2_l8_4gb.json"),
       (3, "qwen3-30b-a3b", 8e9, 1024, 256, 1, "r01_bench_cfg3_q30_8gb.json"),
       (4, "llama3.1-8b", 8e9, 512, 128, 32, "r01_bench_cfg4_l8_batch32_8gb.json"),
       (5, "llama3.3-70b", 24e9, 4096, 128, 1, "r01_bench_cfg5_l70_24gb.json")]
for n, model, budget, prompt, gen, batch, f in CFG:
    spec = catalog.builtin_model(model)
    budget = budget or 0.5 * total_model_bytes(spec)
    bench = json.load(open(os.path.join("profiles", f)))
    row = {"config": n, "model": model, "bench_decode_ms": bench["ms_per_step"],
           "bench_prefill_ms": bench["prefill_passes"][0]["ms"]}
    dt, pt = bench["config"]["decode_tier"], bench["prefill_passes"][0]["tier"]
    for name, db in dbs.items():
        plans = reachable_tiers(spec, m, db, budget, prompt + gen, batch)
        row[f"{name}_decode_ms"] = round(plans[dt].estimated_time * 1e3, 2)
        row[f"{name}_prefill_ms"] = round(plans[pt].estimated_time * 1e3, 2)
    print(json.dumps(row))
