"""`shardplan.simulator` -> `paper_2604_26334_b200.planning.pipeline_model` (drop-in shim)."""
from paper_2604_26334_b200.planning.pipeline_model import *  # noqa: F401,F403
from paper_2604_26334_b200.planning import pipeline_model as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
