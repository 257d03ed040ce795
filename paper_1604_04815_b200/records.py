"""Benchmark records in the reference's schema (chainscan/bench.py:38-74,
:215-231) and the command line's result check.

``CSV_COLUMNS`` is the reference's pinned column list (test_bench_cli.py:27-32);
``EXTENDED_COLUMNS`` appends the device measurements (SURVEY §5 metrics row).

``host_check`` is the reference's validation rule (bench.py:95-114), run on
the host after timing, with numpy — a checker, not a compute path: the
sequential fold (``ufunc.accumulate`` with the dtype pinned, wrapping) is
the reference; integers and max/min must match it exactly — compared as raw
bits, so a wrong sign of zero or a wrong NaN payload fails (the reference's
``np.array_equal`` would let a -0/+0 swap through and reject every NaN) —
and float add must lie inside ``FLOAT_EPS_REL * cumsum|x|`` of it.
"""

from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field
from typing import Optional, Sequence

CSV_COLUMNS = [
    "algorithm", "dtype", "op", "n", "workers", "warp_width", "k",
    "warps_per_block", "runs", "best_seconds", "mean_seconds", "geps",
    "validated", "in_place",
]
EXTENDED_COLUMNS = CSV_COLUMNS + ["device", "timing", "bytes_moved", "gbs", "roofline_frac",
                                  "roofline_denominator_gbs", "impl"]

FLOAT_EPS_REL = {"f32": 1e-5, "f64": 1e-12}


@dataclass
class BenchRecord:
    algorithm: str
    dtype: str
    op: str
    n: int
    workers: int
    warp_width: int
    k: int
    warps_per_block: int
    runs: int
    best_seconds: float
    mean_seconds: float
    geps: float
    validated: str  # "true" | "false" | "skipped"
    in_place: str   # "true" | "false"
    failure: Optional[str] = None  # validation detail, not a column
    extra: dict = field(default_factory=dict)

    def to_row(self, columns=CSV_COLUMNS) -> list:
        return [getattr(self, c) if hasattr(self, c) else self.extra.get(c) for c in columns]

    def to_dict(self, columns=CSV_COLUMNS) -> dict:
        return dict(zip(columns, self.to_row(columns)))


def write_records(records: Sequence[BenchRecord], stream, fmt: str = "csv", extended: bool = False) -> None:
    cols = EXTENDED_COLUMNS if extended else CSV_COLUMNS
    if fmt == "csv":
        w = csv.writer(stream)
        w.writerow(cols)
        for r in records:
            w.writerow(r.to_row(cols))
    elif fmt == "json":
        json.dump([r.to_dict(cols) for r in records], stream, indent=2)
        stream.write("\n")
    else:
        raise ValueError(f"unknown format {fmt!r}")


def format_records(records: Sequence[BenchRecord], fmt: str = "csv", extended: bool = False) -> str:
    buf = io.StringIO()
    write_records(records, buf, fmt, extended)
    return buf.getvalue()


def host_check(x, y, op: str = "add", exclusive: bool = False) -> Optional[str]:
    """None if y (host array) is the scan of x under the reference's rule
    (bench.py:95-114, bit-exact for integers and max/min), else a message
    in the reference's format."""
    import numpy as np
    x = np.asarray(x)
    y = np.asarray(y)
    if y.shape != x.shape:
        return f"shape mismatch {y.shape} vs {x.shape}"
    n = x.size
    if n == 0:
        return None
    uf = {"add": np.add, "max": np.maximum, "min": np.minimum}[op]
    with np.errstate(over="ignore", invalid="ignore"):
        ref = uf.accumulate(x, dtype=x.dtype)
    if exclusive:
        from .operators import make_operator
        ident = make_operator(op, x.dtype).identity
        ref = np.concatenate([np.array([ident], dtype=x.dtype), ref[:-1]])
    if x.dtype.kind == "i" or op in ("max", "min"):
        ub = np.uint32 if x.dtype.itemsize == 4 else np.uint64
        bad = np.nonzero(ref.view(ub) != y.view(ub))[0]
        if bad.size == 0:
            return None
        j = int(bad[0])
        return (f"validation failed at index {j}/{n}: expected {ref[j]!r}, got {y[j]!r} "
                f"(bits {int(ref.view(ub)[j]):#x} vs {int(y.view(ub)[j]):#x}; {bad.size} mismatches)")
    xs = x[:-1] if exclusive else x
    env = FLOAT_EPS_REL["f32" if x.dtype.itemsize == 4 else "f64"] * np.add.accumulate(np.abs(xs, dtype=np.float64))
    if exclusive:
        env = np.concatenate([[0.0], env])
    err = np.abs(y.astype(np.float64) - ref.astype(np.float64))
    bad = np.nonzero(~(err <= env))[0]  # a NaN error is out of the envelope
    if bad.size == 0:
        return None
    j = int(bad[0])
    return (f"validation failed at index {j}/{n}: |{y[j]!r} - {ref[j]!r}| = {err[j]:.3e} > tol {env[j]:.3e} "
            f"({bad.size} indices out of envelope)")
