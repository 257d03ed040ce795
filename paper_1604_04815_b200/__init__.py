"""paper_1604_04815_b200 — B200-native single-pass sum-scan (LightScan, arXiv 1604.04815).

A drop-in for the reference ``chainscan`` package's scan entry point
(``chained_scan``, chainscan/chained.py:316) for the sum operator over
Int32/Int64/Float/Double, plus the derived exclusive scan.  The compute is a
hand-written sm_100a persistent kernel behind the C ABI of ``include/lscan.h``;
Python only moves pointers and streams.

Levels:
  operators / problem / errors   the reference's operator, problem and error surface
  chained                        numpy drop-in: chained_scan(problem, config) -> ndarray
  scan                           torch CUDA tensors: inclusive_scan / exclusive_scan / reduce_sum
  distributed                    one process per GPU, sharded scan with a one-scalar carry exchange
"""

from .operators import (
    DTYPES,
    OPERATOR_NAMES,
    ScanOperator,
    UnsupportedOperatorError,
    dtype_token,
    make_operator,
    parse_dtype,
)
from .problem import ScanProblem, ShapeError
from .errors import DeviceError, LivenessError, ProtocolViolation, WorkspaceError
from .chained import (
    ALGORITHMS,
    ChainConfig,
    SpinPolicy,
    chained_exclusive_scan,
    chained_scan,
    default_worker_count,
    run_algorithm,
)

__version__ = "0.1.0"


def __getattr__(name):
    # torch-level API loaded lazily so the numpy surface imports without torch
    if name in ("inclusive_scan", "exclusive_scan", "reduce", "reduce_sum", "carry_from_totals", "query_config",
                "release_workspaces"):
        from . import scan
        return getattr(scan, name)
    raise AttributeError(name)


__all__ = [
    "ALGORITHMS", "ChainConfig", "DTYPES", "DeviceError", "LivenessError", "OPERATOR_NAMES",
    "ProtocolViolation", "ScanOperator", "ScanProblem", "ShapeError", "SpinPolicy",
    "UnsupportedOperatorError", "WorkspaceError", "chained_exclusive_scan", "chained_scan",
    "default_worker_count", "dtype_token", "make_operator", "parse_dtype", "run_algorithm",
    "inclusive_scan", "exclusive_scan", "reduce", "reduce_sum", "carry_from_totals", "query_config",
    "release_workspaces",
]
