"""Exception types, mirroring the reference's ``hetplan.errors``
(``/root/reference/pkg/src/hetplan/errors.py:4-13``).

When the reference package is importable, these subclass its classes so a
caller's ``except hetplan.errors.NoPath`` also catches ours.
"""
from __future__ import annotations

try:  # pragma: no cover - depends on the host having the reference installed
    from hetplan.errors import NoPath as _RefNoPath
    from hetplan.errors import PlanningError as _RefPlanningError
except Exception:  # noqa: BLE001
    _RefPlanningError = Exception
    _RefNoPath = None


class PlanningError(_RefPlanningError):
    """Base class for all planner errors (errors.py:4-5)."""


if _RefNoPath is not None:  # pragma: no cover
    class NoPath(PlanningError, _RefNoPath):
        """No usable link between two replicas (errors.py:12-13)."""
else:
    class NoPath(PlanningError):
        """No usable link between two replicas (errors.py:12-13)."""


class PartnerLost(NoPath):
    """The other end of a prefill -> decode channel stopped answering: an
    in-kernel doorbell wait was aborted (``PairChannel.abort``) or outlived
    the channel's timeout.  A NoPath: the link to that replica is gone
    (``costs.py:63-64``); the CUDA context and the local KV cache are intact,
    the channel is not (open a new one)."""
