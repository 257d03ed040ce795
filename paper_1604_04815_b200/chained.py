"""Drop-in for the reference scan entry point, on the GPU.

``chained_scan(problem, config=None) -> np.ndarray`` keeps the exact
signature and contract of chainscan's ``chained_scan`` (chained.py:316-357):

* ``problem`` is a ``ScanProblem`` (this package's or the reference's own —
  only ``x``, ``op`` and ``out`` are read); ``op.name`` is ``"add"``,
  ``"max"`` or ``"min"`` (operators.py:111-127);
* the result lands in ``problem.out`` when given (it may alias ``x``, an
  in-place scan) or in a fresh array, and that array object is returned;
* ``n == 0`` returns the (empty) output untouched;
* integers wrap (two's complement) and are bit-identical to the sequential
  oracle, as are max/min for every dtype; float add matches it within the
  reference envelope ``1e-5 / 1e-12 * cumsum|x|`` (bench.py:49, :90-114).

The scan runs on the device through the C ABI (``ls_inclusive_sum_host``):
the host array is streamed through the GPU in chunks with copy-in, scan and
copy-out overlapped.  There is no CPU path.

``ChainConfig`` keeps the reference's fields (chained.py:205-234) and the
drop-in accepts the reference's own ``ChainConfig`` objects.  On the GPU the
worker count and block shape of the parallel scan are decided by the device
(persistent CTAs = co-resident capacity, compile-time tiles), so ``geometry``
and any ``b > 1`` select the same kernel: float add then follows the
reference's B > 1 contract (within the envelope, bench.py:90-114), integers
and max/min are bit-exact regardless.  ``b == 1`` keeps the reference's B = 1
contract — bit-identical to the sequential fold, float add included
(chained.py:290-313; test_acceptance.py:85-111): float add with ``b == 1``
runs the strict left fold on the device (``ls_ordered_scan``: one CTA, one
dependent add per element, ~0.3-0.5 Gelem/s), every other case is already
bit-exact on the parallel kernel.
``spin_budget`` and ``corrupt_slot`` map onto the device watchdog and fault
injection and raise the reference's ``LivenessError``.  ``protocol_checks``
needs no per-call check: every device slot is written once per call by
construction (epoch-tagged words); the explicit device check is
``scan.debug(protocol_checks=True)`` (raises ``ProtocolViolation``).
``on_block`` (a per-block host callback) has no device equivalent and is
rejected.
"""

from __future__ import annotations

import os
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from ._compat import compat
from . import _native as N
from .errors import LivenessError, ProtocolViolation, raise_for_status  # noqa: F401
from .operators import DTYPES, require_device_operator
from .problem import ScanProblem, ShapeError

BLOCK_SCAN_MODES = ("vectorized", "warp-model")
ALGORITHMS = ("chained",)

NP_DT = {np.dtype(np.int32): N.LS_I32, np.dtype(np.int64): N.LS_I64,
         np.dtype(np.float32): N.LS_F32, np.dtype(np.float64): N.LS_F64}


@dataclass(frozen=True)
class SpinPolicy:
    """chained.py:60-82.  The device look-back always spins with a short
    ``nanosleep`` back-off; the policy is validated and kept for parity."""

    kind: str = "spin-yield"
    yield_threshold: int = 1024

    def __post_init__(self):
        if self.kind not in ("spin", "spin-yield"):
            raise ValueError(f"unknown spin policy {self.kind!r}")
        if self.yield_threshold < 1:
            raise ValueError("yield threshold must be >= 1")

    @classmethod
    def spin_then_yield(cls, threshold: int = 1024) -> "SpinPolicy":
        return cls(kind="spin-yield", yield_threshold=threshold)


def default_worker_count() -> int:
    return os.cpu_count() or 1


@dataclass
class ChainConfig:
    """chained.py:205-234 (see module docstring for the GPU meaning)."""

    b: int = field(default_factory=default_worker_count)
    geometry: Optional[object] = None
    spin: SpinPolicy = field(default_factory=SpinPolicy)
    block_scan_mode: str = "vectorized"
    spin_budget: Optional[int] = None
    protocol_checks: bool = True
    corrupt_slot: Optional[int] = None
    on_block: Optional[Callable[[int, int], None]] = None

    def __post_init__(self):
        if self.b < 1:
            raise ValueError(f"worker count must be >= 1, got {self.b}")
        if self.block_scan_mode not in BLOCK_SCAN_MODES:
            raise ValueError(f"unknown block scan mode {self.block_scan_mode!r}; "
                             f"choose from {BLOCK_SCAN_MODES}")


def _device_debug_scan(x: np.ndarray, out: np.ndarray, config: ChainConfig, exclusive: bool,
                       op_name: str) -> None:
    """One device launch over the whole array with the debug hooks armed
    (so that ``corrupt_slot`` names a tile of this array, not of a chunk)."""
    import torch

    from . import scan as S
    with S.debug(spin_budget=int(config.spin_budget or 0),
                 corrupt_tile=-1 if config.corrupt_slot is None else int(config.corrupt_slot)):
        xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
        yd = (S.exclusive_scan if exclusive else S.inclusive_scan)(xd, op=op_name)
        out[...] = yd.cpu().numpy()


def _scan_host(problem, config: Optional[ChainConfig], exclusive: bool) -> np.ndarray:
    op = problem.op
    dtype = require_device_operator(op)
    x = problem.x
    if x.ndim != 1:
        raise compat(ShapeError)(f"input must be 1-D, got shape {x.shape}")
    if x.dtype != dtype:
        # the reference silently computes in x's dtype; the drop-in refuses
        # the mismatch instead of guessing
        raise compat(ShapeError)(f"input dtype {x.dtype} does not match operator dtype {dtype}")
    out = problem.out if problem.out is not None else np.empty_like(x)
    if out.shape != x.shape or out.dtype != dtype:
        raise compat(ShapeError)("out must match the input's shape and dtype")
    if not out.flags.c_contiguous or not out.flags.writeable:
        raise compat(ShapeError)("out must be a writeable C-contiguous array")
    n = x.size
    if n == 0:
        return out
    if config is not None and config.on_block is not None:
        raise ValueError("ChainConfig.on_block is a per-block host callback; the device scan has none")
    if not x.flags.c_contiguous:
        x = np.ascontiguousarray(x)
    if config is not None and (config.spin_budget or config.corrupt_slot is not None):
        _device_debug_scan(x, out, config, exclusive, op.name)
        return out
    # both arrays are contiguous, so overlapping bounds mean real overlap
    aliased = problem.out is not None and np.may_share_memory(out, x)
    if aliased and out.ctypes.data != x.ctypes.data:
        raise compat(ShapeError)("out overlaps x without being the same array (only exact in-place is supported)")
    flags = N.LS_HOST_EXCLUSIVE if exclusive else 0
    if config is not None and config.b == 1 and op.name == "add" and dtype.kind == "f":
        flags |= N.LS_HOST_ORDERED  # the B = 1 bit-exact fold (chained.py:290-313)
    rc = N.lib().ls_scan_host_ex(N.OPS[op.name], NP_DT[dtype], x.ctypes.data, out.ctypes.data, n, flags, -1)
    raise_for_status(rc)
    return out


def chained_scan(problem: ScanProblem, config: Optional[ChainConfig] = None) -> np.ndarray:
    """Inclusive scan of ``problem.x`` under ``problem.op`` (add / max / min)
    on the GPU (chained.py:316-357)."""
    return _scan_host(problem, config, exclusive=False)


def chained_exclusive_scan(problem: ScanProblem, config: Optional[ChainConfig] = None) -> np.ndarray:
    """Exclusive variant (derived mode): y[0] = identity, y[j] = x[0] (+) ... (+) x[j-1]."""
    return _scan_host(problem, config, exclusive=True)


def run_algorithm(name: str, problem: ScanProblem, chain_config: Optional[ChainConfig] = None,
                  rows: Optional[int] = None) -> np.ndarray:
    """bench.py:121-147 dispatch, restricted to the algorithm this package
    provides on the device ("chained")."""
    if name == "chained":
        return chained_scan(problem, chain_config)
    raise ValueError(f"unknown algorithm {name!r}; this package provides {ALGORITHMS}")


__all__ = ["ChainConfig", "SpinPolicy", "chained_scan", "chained_exclusive_scan", "run_algorithm",
           "default_worker_count", "BLOCK_SCAN_MODES", "ALGORITHMS", "DTYPES"]
