"""Status-code -> exception mapping, mirroring the reference's error classes.

chained.py:48-53 (LivenessError, ProtocolViolation), reference.py:34-35
(ShapeError), operators.py:34-35 (UnsupportedOperatorError).

Drop-in compatibility: a caller written against the reference catches the
reference's own classes (``except chainscan.LivenessError``).  When the
reference package is loaded in the process (``chainscan`` in
``sys.modules`` — a caller that names its classes has imported it), every
error the drop-in raises is an instance of BOTH this package's class and
the reference class of the same name (``compat``), so either ``except``
clause matches.  Nothing here imports the reference.
"""

from __future__ import annotations

from . import _native as N
from ._compat import compat
from .operators import UnsupportedOperatorError
from .problem import ShapeError


class LivenessError(RuntimeError):
    """A debug spin budget ran out while waiting on a slot (chained.py:48-49)."""


class ProtocolViolation(RuntimeError):
    """The write-once slot discipline was broken (chained.py:52-53)."""


class DeviceError(RuntimeError):
    """A CUDA runtime call inside the native library failed."""


class WorkspaceError(RuntimeError):
    """The carry-chain workspace is missing, too small or misaligned."""


def raise_for_status(code: int) -> None:
    if code == N.LS_OK:
        return
    detail = N.last_detail()
    name = N.status_string(code)
    msg = f"{name}: {detail}" if detail else name
    if code == N.LS_ERR_INVALID_ARG:
        raise compat(ShapeError)(msg)
    if code == N.LS_ERR_UNSUPPORTED_DTYPE:
        raise compat(UnsupportedOperatorError)(msg)
    if code == N.LS_ERR_LIVENESS:
        raise compat(LivenessError)(msg)
    if code == N.LS_ERR_PROTOCOL:
        raise compat(ProtocolViolation)(msg)
    if code == N.LS_ERR_WORKSPACE:
        raise WorkspaceError(msg)
    raise DeviceError(msg)
