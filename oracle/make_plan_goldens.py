"""Generate tests/golden/plan_goldens.json from the UNMODIFIED reference planner.

Test infrastructure (ORACLE). Run in the build container, where
/root/reference exists:  python oracle/make_plan_goldens.py
Reference presets are read from the reference's own data files
(`pkg/src/shardplan/data/{models,machines}/*.json`), so the drop-in
catalog's restated values are checked too; B200 presets come from this
build's catalog. Each case stores the full model/machine dicts, so the
parity test needs nothing but this file.
"""

import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)
REF_DATA = "/root/reference/pkg/src/shardplan/data"

from paper_2604_26334_b200.planning import catalog  # noqa: E402
from paper_2604_26334_b200.planning.graph import model_from_dict, total_model_bytes  # noqa: E402

GB = 1e9


def ref_doc(kind, name):
    with open(os.path.join(REF_DATA, kind, name + ".json")) as fh:
        return json.load(fh)


def cases():
    out = []

    def add(model_doc, machine_doc, budget, context, batch=1, tier=None, tag=""):
        out.append({"id": len(out), "tag": tag, "model": model_doc, "machine": machine_doc,
                    "budget": budget, "context": context, "batch": batch, "tier": tier})

    # A. reference presets x reference machines
    for model in ("nemo4b", "nemo8b", "qwen30b", "qwen235b", "cr1"):
        for machine in ("laptop", "desktop", "workstation"):
            for budget in (2, 4, 8, 16):
                for ctx in (4096, 16384):
                    add(ref_doc("models", model), ref_doc("machines", machine), budget * GB,
                        ctx, tag=f"{model}/{machine}/{budget}G/ctx{ctx}")
    for batch in (4, 64):
        for budget in (4, 16):
            add(ref_doc("models", "nemo8b"), ref_doc("machines", "workstation"), budget * GB,
                1024, batch, tag=f"nemo8b/workstation/{budget}G/ctx1024/b{batch}")
    # B. SURVEY Appendix B goldens (workstation, ctx 4096)
    for model in ("nemo8b", "qwen30b"):
        for budget in (2, 4, 8, 16, 32):
            add(ref_doc("models", model), ref_doc("machines", "workstation"), budget * GB, 4096,
                tag=f"appendixB/{model}/{budget}G")
    # C. BASELINE.json configs on the b200 preset
    b200 = catalog.machine_doc("b200")
    add(catalog.model_doc("llama3.1-8b"), b200, 4 * GB, 2048 + 256, tag="cfg2/L8@4G")
    add(catalog.model_doc("qwen3-30b-a3b"), b200, 8 * GB, 1024 + 256, tag="cfg3/Q30@8G")
    add(catalog.model_doc("llama3.1-8b"), b200, 8 * GB, 512 + 128, 32, tag="cfg4/L8b32@8G")
    add(catalog.model_doc("llama3.3-70b"), b200, 24 * GB, 4096 + 128, tag="cfg5/L70@24G")
    tiny = catalog.model_doc("tiny-llama")
    tiny_budget = 0.5 * total_model_bytes(model_from_dict(tiny))
    add(tiny, b200, tiny_budget, 128 + 32, tag="cfg1/tiny@50%")
    for tier in (1, 4, 16, 32, 64, 512, 1024, 2048, 4096, 8192, 16384):
        add(tiny, b200, tiny_budget, 128 + 32, tier=tier, tag=f"cfg1/tiny@50%/tier{tier}")
    for tier in (1, 2048):
        add(catalog.model_doc("llama3.1-8b"), b200, 4 * GB, 2048 + 256, tier=tier,
            tag=f"cfg2/L8@4G/tier{tier}")
    # D. error contract
    add(ref_doc("models", "qwen235b"), ref_doc("machines", "workstation"), 1 * GB, 16384,
        tag="err/budget-below-floor")
    add(ref_doc("models", "nemo8b"), ref_doc("machines", "desktop"), 20 * GB, 4096,
        tag="err/budget-over-vram")
    return out


def main():
    cfgs = cases()
    proc = subprocess.run([sys.executable, os.path.join(HERE, "plan_oracle.py")],
                          input=json.dumps(cfgs), capture_output=True, text=True, check=True)
    results = {r["id"]: r for r in json.loads(proc.stdout)}
    for c in cfgs:
        r = results[c["id"]]
        c["expect"] = {k: r[k] for k in ("sha256", "error") if k in r}
        c["oracle_seconds"] = round(r["seconds"], 4)
    dest = os.path.join(REPO, "tests", "golden", "plan_goldens.json")
    with open(dest, "w") as fh:
        json.dump({"generator": "oracle/make_plan_goldens.py",
                   "reference": "/root/reference/pkg/src/shardplan (unmodified)",
                   "cases": cfgs}, fh, indent=1, sort_keys=True)
        fh.write("\n")
    print(f"wrote {len(cfgs)} cases to {dest}")


if __name__ == "__main__":
    main()
