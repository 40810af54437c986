"""ORACLE (test infrastructure only): the reference planner, run as-is.

Imports the UNMODIFIED reference `shardplan` package — from
/root/reference/pkg/src when present (this container), else from the
pip-installed copy in baseline/_ref (travels to the GPU box) — and prints,
for each requested configuration, the sha256 of the exact bytes
`save_table` writes (`pkg/src/shardplan/planner.py:527-530`) or the
exception it raises (type, budget_bytes, required_bytes, what).

Only tests/ and bench.py's cpu_baseline leg run this file, always as a
separate process (the reference and the drop-in shim share the package
name `shardplan`). Usage:  python oracle/plan_oracle.py < configs.json
"""

import hashlib
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def reference_path() -> str:
    for cand in ("/root/reference/pkg/src", os.path.join(REPO, "baseline", "_ref")):
        if os.path.isdir(os.path.join(cand, "shardplan")):
            return cand
    raise SystemExit("reference shardplan not found (neither /root/reference nor baseline/_ref)")


sys.path.insert(0, reference_path())
sys.dont_write_bytecode = True

from shardplan import planner as P  # noqa: E402  (the reference)
from shardplan.machine import machine_from_dict  # noqa: E402
from shardplan.model_graph import model_from_dict  # noqa: E402
from shardplan.profile_db import synth_profile  # noqa: E402
from shardplan.errors import InfeasibleBudget, InfeasibleSchedule  # noqa: E402


def run(cfgs):
    dbs = {}
    out = []
    for cfg in cfgs:
        model = model_from_dict(cfg["model"])
        machine = machine_from_dict(cfg["machine"])
        key = json.dumps(cfg["machine"], sort_keys=True)
        if key not in dbs:
            dbs[key] = synth_profile(machine)
        db = dbs[key]
        t0 = time.perf_counter()
        rec = {"id": cfg["id"]}
        try:
            if cfg.get("tier") is not None:
                _, _, _, plans = P.plan_tier(model, machine, db, cfg["budget"], cfg["context"],
                                             cfg["tier"], cfg.get("batch", 1))
                sel = P.select_plan(plans)
                doc = [P._plan_to_dict(p) for p in plans] + [P._plan_to_dict(sel)]
                blob = json.dumps(doc, indent=2, sort_keys=True) + "\n"
            else:
                table = P.build_tier_table(model, machine, db, cfg["budget"], cfg["context"],
                                           kv_replicas=cfg.get("batch", 1))
                blob = json.dumps(P.table_to_dict(table), indent=2, sort_keys=True) + "\n"
            rec["sha256"] = hashlib.sha256(blob.encode()).hexdigest()
        except (InfeasibleBudget, InfeasibleSchedule) as exc:
            rec["error"] = {"type": type(exc).__name__,
                            "budget_bytes": getattr(exc, "budget_bytes", None),
                            "required_bytes": getattr(exc, "required_bytes", None),
                            "what": getattr(exc, "what", None), "message": str(exc)}
        rec["seconds"] = time.perf_counter() - t0
        out.append(rec)
    return out


if __name__ == "__main__":
    json.dump(run(json.load(sys.stdin)), sys.stdout)
