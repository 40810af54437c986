"""Plan parity: this build's planner vs the UNMODIFIED reference planner.

Golden fixtures (tests/golden/plan_goldens.json) hold, per configuration,
the sha256 of the exact bytes the reference's `save_table` writes
(`pkg/src/shardplan/planner.py:527-530`), or the exception it raised, as
produced by oracle/make_plan_goldens.py. Bit-exact equality is required.
"""

import hashlib
import json
import os

import pytest

from paper_2604_26334_b200.planning import (InfeasibleBudget, InfeasibleSchedule,
                                            build_tier_table, machine_from_dict,
                                            model_from_dict, plan_tier, select_plan,
                                            synth_profile, table_to_dict)
from paper_2604_26334_b200.planning.placement import _plan_doc
from paper_2604_26334_b200.planning.hardware import machine_to_dict

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = json.load(open(os.path.join(HERE, "golden", "plan_goldens.json")))
_DBS = {}


def _db(machine):
    key = json.dumps(machine_to_dict(machine), sort_keys=True)
    if key not in _DBS:
        _DBS[key] = synth_profile(machine)
    return _DBS[key]


def mine(case):
    model = model_from_dict(case["model"])
    machine = machine_from_dict(case["machine"])
    db = _db(machine)
    try:
        if case.get("tier") is not None:
            _, _, _, plans = plan_tier(model, machine, db, case["budget"], case["context"],
                                       case["tier"], case["batch"])
            doc = [_plan_doc(p) for p in plans] + [_plan_doc(select_plan(plans))]
        else:
            doc = table_to_dict(build_tier_table(model, machine, db, case["budget"],
                                                 case["context"], kv_replicas=case["batch"]))
        blob = json.dumps(doc, indent=2, sort_keys=True) + "\n"
        return {"sha256": hashlib.sha256(blob.encode()).hexdigest()}
    except (InfeasibleBudget, InfeasibleSchedule) as exc:
        return {"error": {"type": type(exc).__name__,
                          "budget_bytes": getattr(exc, "budget_bytes", None),
                          "required_bytes": getattr(exc, "required_bytes", None),
                          "what": getattr(exc, "what", None), "message": str(exc)}}


@pytest.mark.parametrize("case", GOLDEN["cases"], ids=[c["tag"] for c in GOLDEN["cases"]])
def test_plan_bit_exact(case):
    assert mine(case) == case["expect"]


def test_appendix_b_digests_match_survey():
    # sha256[:16] of the workstation ctx-4096 tables.
    want = {"nemo8b/2G": "2439928456e689fd", "nemo8b/4G": "51d37f77ec9869bd",
            "nemo8b/8G": "4d2b4d9faea509d7", "nemo8b/16G": "53315fb9c725be64",
            "nemo8b/32G": "c6b764857beac7b9", "qwen30b/2G": "a6d526eb7e30435b",
            "qwen30b/4G": "55b2090246246601", "qwen30b/8G": "ba55ed5fc9832d75",
            "qwen30b/16G": "709937c73bf104e5", "qwen30b/32G": "85331f3b3448ed36"}
    got = {c["tag"][len("appendixB/"):]: mine(c)["sha256"][:16]
           for c in GOLDEN["cases"] if c["tag"].startswith("appendixB/")}
    assert got == want
