"""`shardplan.errors` -> `paper_2604_26334_b200.planning.faults` (drop-in shim)."""
from paper_2604_26334_b200.planning.faults import *  # noqa: F401,F403
from paper_2604_26334_b200.planning import faults as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
