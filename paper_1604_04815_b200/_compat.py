"""Reference-compatible exception classes (see errors.py).

When the reference package is loaded in the process (``chainscan`` in
``sys.modules``), ``compat(cls)`` returns a subclass of both ``cls`` and the
reference's class of the same name, so a caller's ``except
chainscan.ShapeError`` (etc.) matches what the drop-in raises.  Nothing here
imports the reference.
"""

from __future__ import annotations

import sys
import threading


# reference module that defines each mirrored class
_REF_HOME = {
    "ShapeError": "chainscan.reference",
    "UnsupportedOperatorError": "chainscan.operators",
    "LivenessError": "chainscan.chained",
    "ProtocolViolation": "chainscan.chained",
}
_compat_cache: dict = {}
_compat_lock = threading.Lock()


def compat(cls: type) -> type:
    """``cls``, or — when the reference package is loaded — a subclass of
    both ``cls`` and the reference's class of the same name."""
    home = _REF_HOME.get(cls.__name__)
    mod = sys.modules.get(home) if home else None
    ref = getattr(mod, cls.__name__, None) if mod is not None else None
    if not isinstance(ref, type) or not issubclass(ref, BaseException) or issubclass(cls, ref):
        return cls
    key = (cls, ref)
    with _compat_lock:
        c = _compat_cache.get(key)
        if c is None:
            c = type(cls.__name__, (cls, ref), {"__module__": cls.__module__, "__doc__": cls.__doc__})
            _compat_cache[key] = c
    return c
