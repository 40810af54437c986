"""`shardplan.cli` -> `paper_2604_26334_b200.planning.command` (drop-in shim)."""
from paper_2604_26334_b200.planning.command import *  # noqa: F401,F403
from paper_2604_26334_b200.planning import command as _impl

globals().update({k: v for k, v in vars(_impl).items() if not k.startswith("__")})

if __name__ == "__main__":
    import sys
    sys.exit(main())
