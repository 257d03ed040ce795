"""Benchmark records in the reference's schema (chainscan/bench.py:38-74,
:215-231) and an on-device result check for the command line.

``CSV_COLUMNS`` is the reference's pinned column list (test_bench_cli.py:27-32);
``EXTENDED_COLUMNS`` appends the device measurements (SURVEY §5 metrics row).

``device_check`` validates a device scan without any CPU scan: integers by
the exact difference identity y[0] = x[0], y[j] - y[j-1] = x[j] (two's
complement), max/min against ``torch.cummax``/``cummin`` (exact), float add
against a float64 device cumsum within the reference envelope
``FLOAT_EPS_REL * cumsum|x|`` (bench.py:49, :90-114).
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


def device_check(x, y, op: str = "add", exclusive: bool = False) -> Optional[str]:
    """None if the device result y is the scan of x, else a message."""
    import torch
    n = x.numel()
    if y.shape != x.shape:
        return f"shape mismatch {tuple(y.shape)} vs {tuple(x.shape)}"
    if n == 0:
        return None
    if exclusive:
        # exclusive y is the inclusive scan shifted right by one
        x, y = x[:-1], y[1:]
        n -= 1
        if n == 0:
            return None
    if op in ("max", "min"):
        ref = (torch.cummax if op == "max" else torch.cummin)(x, 0).values
        bad = torch.nonzero(~((ref == y) | (torch.isnan(ref) & torch.isnan(y))))
    elif not x.dtype.is_floating_point:
        d = torch.empty_like(x)
        d[0] = y[0]
        d[1:] = y[1:] - y[:-1]  # wraps like the scan itself
        bad = torch.nonzero(d != x)
    else:
        ref = torch.cumsum(x.double(), 0)
        tol = FLOAT_EPS_REL["f32" if x.dtype == torch.float32 else "f64"] * torch.cumsum(x.double().abs(), 0)
        bad = torch.nonzero((y.double() - ref).abs() > tol)
    if bad.numel() == 0:
        return None
    j = int(bad[0, 0])
    return f"validation failed at index {j}/{n}: {bad.shape[0]} mismatches"
