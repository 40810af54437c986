"""`shardplan.kernels` -> `paper_2604_26334_b200.planning.vocab` (drop-in shim)."""
from paper_2604_26334_b200.planning.vocab import *  # noqa: F401,F403
from paper_2604_26334_b200.planning import vocab as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})
