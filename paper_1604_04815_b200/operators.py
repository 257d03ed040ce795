"""Element types and the scan operator — the reference's operator surface.

Mirrors ``chainscan.operators`` (operators.py:24-127): the same dtype tokens,
the same ``make_operator(name, elem_type)`` factory and error class, and an
operator object exposing ``name``, ``dtype`` and ``identity``.  The device
kernels implement all three operators of the reference's table: ``add`` (the
north-star operator), ``max`` and ``min``; float max/min propagate NaN like
``np.maximum`` / ``np.minimum``.

Integer add wraps modulo 2^width (two's complement), as the reference's
``np.add`` under ``errstate(over="ignore")`` does (operators.py:74-100).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._compat import compat

# operators.py:24-29
DTYPES = {
    "i32": np.dtype(np.int32),
    "i64": np.dtype(np.int64),
    "f32": np.dtype(np.float32),
    "f64": np.dtype(np.float64),
}

OPERATOR_NAMES = ("add", "max", "min")
DEVICE_OPERATORS = ("add", "max", "min")


class UnsupportedOperatorError(ValueError):
    """Unknown operator name or element type token (operators.py:34-35)."""


def parse_dtype(token) -> np.dtype:
    """Map an element-type token (i32/i64/f32/f64) to its numpy dtype (operators.py:38-47)."""
    if isinstance(token, np.dtype):
        if token in DTYPES.values():
            return token
        raise compat(UnsupportedOperatorError)(f"unsupported element type {token}")
    try:
        return DTYPES[token]
    except (KeyError, TypeError):
        raise compat(UnsupportedOperatorError)(
            f"unknown element type {token!r}; supported: {', '.join(DTYPES)}") from None


def dtype_token(dtype) -> str:
    dtype = np.dtype(dtype)
    for tok, dt in DTYPES.items():
        if dt == dtype:
            return tok
    raise compat(UnsupportedOperatorError)(f"no token for dtype {dtype}")


@dataclass(frozen=True)
class ScanOperator:
    """An associative operator bound to an element dtype (operators.py:58-72)."""

    name: str
    dtype: np.dtype
    identity: object

    def apply(self, a, b):
        with np.errstate(over="ignore"):
            if self.name == "add":
                return self.dtype.type(np.add(self.dtype.type(a), self.dtype.type(b)))
            if self.name == "max":
                return self.dtype.type(np.maximum(a, b))
            return self.dtype.type(np.minimum(a, b))


def make_operator(name: str, elem_type) -> ScanOperator:
    """operators.py:111-127: add (identity 0), max, min."""
    dtype = parse_dtype(elem_type)
    if name == "add":
        identity = dtype.type(0)
    elif name == "max":
        identity = dtype.type(np.iinfo(dtype).min if dtype.kind == "i" else -np.inf)
    elif name == "min":
        identity = dtype.type(np.iinfo(dtype).max if dtype.kind == "i" else np.inf)
    else:
        raise compat(UnsupportedOperatorError)(
            f"unknown operator {name!r}; supported: {', '.join(OPERATOR_NAMES)}")
    return ScanOperator(name=name, dtype=dtype, identity=identity)


def require_device_operator(op) -> np.dtype:
    """The operator must be one the device implements (add / max / min)."""
    name = getattr(op, "name", None)
    if name not in DEVICE_OPERATORS:
        raise compat(UnsupportedOperatorError)(
            f"operator {name!r} has no device scan; supported: {', '.join(DEVICE_OPERATORS)}")
    return parse_dtype(np.dtype(op.dtype))
