"""Error contract of the planning API.

Mirrors the exception hierarchy the reference exposes at
`pkg/src/shardplan/errors.py:4-35` so callers can catch the same types:
a base `ShardPlanError`, `SpecError` for invalid inputs, `InfeasibleBudget`
carrying (budget_bytes, required_bytes, what), `InfeasibleSchedule` for
budgets or plans that exceed VRAM, and `FormatError` for persisted files.
"""

from __future__ import annotations

__all__ = ["ShardPlanError", "SpecError", "InfeasibleBudget",
           "InfeasibleSchedule", "FormatError"]


class ShardPlanError(Exception):
    """Root of every planner / executor error raised by this package."""


class SpecError(ShardPlanError):
    """An input spec (model, machine, request) breaks an invariant."""


class InfeasibleBudget(ShardPlanError):
    """The VRAM budget cannot hold the minimum working set.

    The message text follows the reference (`errors.py:20-27`): the CLI
    tests grep for "short".
    """

    def __init__(self, budget_bytes: float, required_bytes: float, what: str = "scratch"):
        self.budget_bytes = budget_bytes
        self.required_bytes = required_bytes
        self.what = what
        missing_mb = (required_bytes - budget_bytes) / 1e6
        super().__init__(
            "VRAM budget %.1f MB is short %.1f MB of the %.1f MB needed for %s"
            % (budget_bytes / 1e6, missing_mb, required_bytes / 1e6, what))


class InfeasibleSchedule(ShardPlanError):
    """A plan (or the budget itself) does not fit the device's VRAM."""


class FormatError(ShardPlanError):
    """Unknown version tag or malformed body in a persisted artifact."""
