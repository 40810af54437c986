"""Placement planner of the pipelined-sharding path (pure Python, bit-exact
with the reference `shardplan` package)."""

from .faults import *  # noqa: F401,F403
from .vocab import *  # noqa: F401,F403
from .hardware import *  # noqa: F401,F403
from .graph import *  # noqa: F401,F403
from .costdb import *  # noqa: F401,F403
from .placement import *  # noqa: F401,F403
from .pipeline_model import *  # noqa: F401,F403
from .catalog import *  # noqa: F401,F403
