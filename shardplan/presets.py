"""`shardplan.presets` -> `paper_2604_26334_b200.planning.catalog` (drop-in shim)."""
from paper_2604_26334_b200.planning.catalog import *  # noqa: F401,F403
from paper_2604_26334_b200.planning import catalog as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
