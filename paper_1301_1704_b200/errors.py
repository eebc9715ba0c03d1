"""Exception types of the drop-in API (reference: pkg/src/fmmkit/errors.py:4-21).

When the reference package `fmmkit` is already imported in the process (i.e.
this framework is being used as its backend), each class also derives from
the reference class of the same name, so `except fmmkit.errors.DomainError`
and `pytest.raises(fmmkit.CapacityError)` keep working unchanged.  Nothing
here imports the reference.
"""

from __future__ import annotations

import sys

_ref = sys.modules.get("fmmkit.errors")


def _bases(name: str, *own: type) -> tuple[type, ...]:
    ref_cls = getattr(_ref, name, None) if _ref is not None else None
    if ref_cls is None:
        return own
    return tuple(b for b in own if not issubclass(ref_cls, b)) + (ref_cls,)


class FmmError(*_bases("FmmError", Exception)):  # errors.py:4
    """Base class for all errors of the B200 build."""


class CapacityError(*_bases("CapacityError", FmmError)):  # errors.py:8
    """A configured resource limit (level cap, histogram budget, integer width) was exceeded."""


class DomainError(*_bases("DomainError", FmmError, ValueError)):  # errors.py:12
    """An argument violated a documented precondition."""


class RoutingError(*_bases("RoutingError", FmmError)):  # errors.py:16
    """Multi-GPU exchange could not deliver a box it was asked for."""


class InfeasiblePartitionError(*_bases("InfeasiblePartitionError", FmmError)):  # errors.py:20
    """More ranks were requested than there are non-empty boxes to assign."""


class NativeError(FmmError, RuntimeError):
    """The CUDA library failed (or is missing on a GPU host)."""
