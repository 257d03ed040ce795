"""Device-level API on torch CUDA tensors (the B200 hot path).

``inclusive_scan`` / ``exclusive_scan`` / ``reduce_sum`` call the C ABI of
``include/lscan.h`` with raw device pointers and the current CUDA stream;
torch is only the allocator and stream plumbing.  Each (device, stream) keeps
one workspace (the carry-chain slot buffer), zeroed once and then reused
across calls through its epoch tags.

Reference counterpart: ``chained_scan`` (chainscan/chained.py:316-357) with
op ``add``; the numpy-level drop-in with the reference's exact signature is
``paper_1604_04815_b200.chained.chained_scan``.
"""

from __future__ import annotations

import threading
from collections import OrderedDict
from typing import Dict, Optional, Tuple

import torch

from ._compat import compat
from . import _native as N
from .errors import raise_for_status
from .operators import UnsupportedOperatorError
from .problem import ShapeError

TORCH_DT = {
    torch.int32: N.LS_I32,
    torch.int64: N.LS_I64,
    torch.float32: N.LS_F32,
    torch.float64: N.LS_F64,
}

_ws_lock = threading.Lock()
# (device index, raw stream) -> workspace, least recently created first.  A
# caller cycling through many streams would otherwise keep one buffer per
# stream forever: beyond _WS_CACHE entries the oldest is dropped (the caching
# allocator hands its memory back only to work ordered after it on the stream
# it was allocated on, so a scan still in flight there is unaffected).
_WS_CACHE = 64
_workspaces: "OrderedDict[Tuple[int, int], torch.Tensor]" = OrderedDict()


def dtype_code(dtype: torch.dtype) -> int:
    try:
        return TORCH_DT[dtype]
    except KeyError:
        raise compat(UnsupportedOperatorError)(
            f"unsupported element type {dtype}; supported: int32, int64, float32, float64") from None


def workspace(device: torch.device, stream: torch.cuda.Stream, nbytes: int) -> torch.Tensor:
    """The (device, stream)'s workspace, grown (and zeroed) on demand."""
    key = (device.index, stream.cuda_stream)
    with _ws_lock:
        ws = _workspaces.get(key)
        if ws is None or ws.numel() < nbytes:
            size = max(nbytes, 1 << 20)
            if ws is not None:
                size = max(size, 2 * ws.numel())
            with torch.cuda.stream(stream):
                ws = torch.empty(size + 128, dtype=torch.uint8, device=device)
                # 128-byte alignment of the header line
                off = (-ws.data_ptr()) % 128
                ws = ws[off:off + size]
                raise_for_status(N.lib().ls_workspace_init(ws.data_ptr(), ws.numel(), stream.cuda_stream))
            _workspaces[key] = ws
            while len(_workspaces) > _WS_CACHE:
                _workspaces.popitem(last=False)
        return ws


def release_workspaces(device: Optional[torch.device] = None) -> int:
    """Drop the cached per-stream workspaces (of one device, or all); the
    next scan on a stream allocates and zeroes a fresh one.  Returns how many
    were dropped."""
    with _ws_lock:
        keys = [k for k in _workspaces if device is None or k[0] == torch.device(device).index]
        for k in keys:
            del _workspaces[k]
    return len(keys)


def _check_1d(x: torch.Tensor, what: str = "input") -> None:
    if not isinstance(x, torch.Tensor):
        raise TypeError(f"{what} must be a torch.Tensor")
    if x.dim() != 1:
        raise compat(ShapeError)(f"{what} must be 1-D, got shape {tuple(x.shape)}")
    if not x.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (there is no CPU path)")


def _scalar_ptr(t: Optional[torch.Tensor], like: torch.Tensor, what: str) -> Optional[int]:
    if t is None:
        return None
    if t.device != like.device or t.dtype != like.dtype or t.numel() < 1:
        raise ValueError(f"{what} must be a device tensor of {like.dtype} on {like.device}")
    return t.data_ptr()


def op_code(op: str) -> int:
    try:
        return N.OPS[op]
    except KeyError:
        raise compat(UnsupportedOperatorError)(f"unknown operator {op!r}; supported: {', '.join(N.OPS)}") from None


# the raw cudaStream_t of a device's current stream, without building a Stream
# object (torch's own accessor, used by its code generators)
try:
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover - older torch
    def _raw_stream(index: int) -> int:
        return torch.cuda.current_stream(index).cuda_stream


_ws_need: Dict[Tuple[int, int], int] = {}


def _ws_bytes(dt: int, n: int) -> int:
    key = (dt, n)
    b = _ws_need.get(key)
    if b is None:
        if len(_ws_need) > 4096:
            _ws_need.clear()
        b = _ws_need[key] = N.lib().ls_workspace_bytes(dt, n)
    return b


_get_device = getattr(torch._C, "_cuda_getDevice", torch.cuda.current_device)


def _scan(x: torch.Tensor, out: Optional[torch.Tensor], carry_in, total_out, exclusive: bool,
          op: str = "add") -> torch.Tensor:
    # the per-call path is kept lean (it is most of the cost of a small scan):
    # integer device indices, raw stream pointers, cached workspace sizes
    if type(x) is not torch.Tensor and not isinstance(x, torch.Tensor):
        raise TypeError("input must be a torch.Tensor")
    if x.dim() != 1:
        raise compat(ShapeError)(f"input must be 1-D, got shape {tuple(x.shape)}")
    if not x.is_cuda:
        raise ValueError("input must be a CUDA tensor (there is no CPU path)")
    dt = TORCH_DT.get(x.dtype)
    if dt is None:
        dtype_code(x.dtype)  # raises UnsupportedOperatorError
    oc = N.OPS.get(op)
    if oc is None:
        op_code(op)  # raises UnsupportedOperatorError
    idx = x.get_device()
    n = x.numel()
    if out is None:
        out = torch.empty_like(x, memory_format=torch.contiguous_format)
    elif out is not x:
        _check_1d(out, "out")
        if out.numel() != n:
            raise compat(ShapeError)("out shape must match input shape")
        if out.dtype != x.dtype or out.get_device() != idx:
            raise ValueError("out must have the input's dtype and device")
        if not out.is_contiguous():
            raise compat(ShapeError)("out must be contiguous")
    if not x.is_contiguous():
        if out is x:
            raise compat(ShapeError)("in-place scan needs a contiguous tensor")
        x = x.contiguous()
    prev = _get_device()
    switch = idx != prev
    if switch:
        torch.cuda.set_device(idx)
    try:
        sp = _raw_stream(idx)
        ws = _workspaces.get((idx, sp))
        need = _ws_bytes(dt, n)
        if ws is None or ws.numel() < need:
            ws = workspace(x.device, torch.cuda.current_stream(x.device), need)
        L = N.lib()
        fn = L.ls_exclusive_scan if exclusive else L.ls_inclusive_scan
        rc = fn(oc, dt, x.data_ptr() if n else None, out.data_ptr() if n else None, n,
                None if carry_in is None else _scalar_ptr(carry_in, x, "carry_in"),
                None if total_out is None else _scalar_ptr(total_out, x, "total_out"),
                ws.data_ptr(), ws.numel(), sp)
    finally:
        if switch:
            torch.cuda.set_device(prev)
    if rc:
        raise_for_status(rc)
    return out


def inclusive_scan(x: torch.Tensor, out: Optional[torch.Tensor] = None, *,
                   carry_in: Optional[torch.Tensor] = None,
                   total_out: Optional[torch.Tensor] = None, op: str = "add") -> torch.Tensor:
    """y[j] = carry (+) x[0] (+) ... (+) x[j] on the device; ``out`` may be ``x``.

    ``op`` is ``"add"`` (default), ``"max"`` or ``"min"``.  ``carry_in`` /
    ``total_out`` are optional one-element device tensors of x's dtype (the
    multi-GPU carry seam)."""
    return _scan(x, out, carry_in, total_out, exclusive=False, op=op)


def exclusive_scan(x: torch.Tensor, out: Optional[torch.Tensor] = None, *,
                   carry_in: Optional[torch.Tensor] = None,
                   total_out: Optional[torch.Tensor] = None, op: str = "add") -> torch.Tensor:
    """y[0] = carry (or the identity), y[j] = carry (+) x[0] (+) ... (+) x[j-1]."""
    return _scan(x, out, carry_in, total_out, exclusive=True, op=op)


def ordered_scan(x: torch.Tensor, out: Optional[torch.Tensor] = None, *, exclusive: bool = False,
                 carry_in: Optional[torch.Tensor] = None, total_out: Optional[torch.Tensor] = None,
                 op: str = "add") -> torch.Tensor:
    """The strict left fold on the device (``ls_ordered_scan``): y[j] =
    y[j-1] (+) x[j] in sequence, bit-identical to the reference's
    ``sequential_scan`` and to its ``ChainConfig(b=1)`` path (chained.py:290-313)
    for every operator, float add included.  One CTA runs the dependent chain
    (an exactness mode at roughly one add latency per element, not a fast
    path); ``inclusive_scan`` is the parallel scan."""
    _check_1d(x)
    dt = dtype_code(x.dtype)
    oc = op_code(op)
    n = x.numel()
    if out is None:
        out = torch.empty_like(x, memory_format=torch.contiguous_format)
    elif out is not x:
        _check_1d(out, "out")
        if out.numel() != n or out.dtype != x.dtype or out.device != x.device or not out.is_contiguous():
            raise compat(ShapeError)("out must be a contiguous tensor of x's shape, dtype and device")
    if not x.is_contiguous():
        if out is x:
            raise compat(ShapeError)("in-place scan needs a contiguous tensor")
        x = x.contiguous()
    stream = torch.cuda.current_stream(x.device)
    with torch.cuda.device(x.device):
        rc = N.lib().ls_ordered_scan(oc, dt, x.data_ptr() if n else None, out.data_ptr() if n else None, n,
                                     1 if exclusive else 0, _scalar_ptr(carry_in, x, "carry_in"),
                                     _scalar_ptr(total_out, x, "total_out"), stream.cuda_stream)
    raise_for_status(rc)
    return out


def reduce(x: torch.Tensor, total_out: Optional[torch.Tensor] = None, op: str = "add") -> torch.Tensor:
    """Deterministic device reduction of x into a one-element tensor."""
    _check_1d(x)
    dt = dtype_code(x.dtype)
    oc = op_code(op)
    if not x.is_contiguous():
        x = x.contiguous()
    if total_out is None:
        total_out = torch.empty(1, dtype=x.dtype, device=x.device)
    stream = torch.cuda.current_stream(x.device)
    L = N.lib()
    ws = workspace(x.device, stream, L.ls_workspace_bytes(dt, 0))
    with torch.cuda.device(x.device):
        rc = L.ls_reduce(oc, dt, x.data_ptr() if x.numel() else None, x.numel(),
                             _scalar_ptr(total_out, x, "total_out"), ws.data_ptr(), ws.numel(),
                             stream.cuda_stream)
    raise_for_status(rc)
    return total_out


def reduce_sum(x: torch.Tensor, total_out: Optional[torch.Tensor] = None) -> torch.Tensor:
    """Deterministic device sum of x into a one-element tensor."""
    return reduce(x, total_out, op="add")


def carry_from_totals(totals: torch.Tensor, rank: int, carry_out: Optional[torch.Tensor] = None,
                      op: str = "add") -> torch.Tensor:
    """carry = totals[0] (+) ... (+) totals[rank-1] on the device (fixed order)."""
    _check_1d(totals, "totals")
    dt = dtype_code(totals.dtype)
    oc = op_code(op)
    if carry_out is None:
        carry_out = torch.empty(1, dtype=totals.dtype, device=totals.device)
    stream = torch.cuda.current_stream(totals.device)
    with torch.cuda.device(totals.device):
        rc = N.lib().ls_carry_from_totals(oc, dt, totals.data_ptr(), totals.numel(), rank,
                                         carry_out.data_ptr(), stream.cuda_stream)
    raise_for_status(rc)
    return carry_out


def query_config(dtype: torch.dtype, n: int) -> dict:
    """Launch geometry the scan uses for (dtype, n) on the current device."""
    import ctypes
    out = (ctypes.c_int64 * 6)()
    raise_for_status(N.lib().ls_query_config(dtype_code(dtype), n, out))
    keys = ("grid", "threads", "tile_elems", "stages", "ctas_per_sm", "sms")
    return dict(zip(keys, (int(v) for v in out)))


def query_multi_config(dtype: torch.dtype, n_local: int) -> dict:
    """The multi-GPU kernel's default grid and tile (the block-cyclic stripe
    is grid x tile elements)."""
    import ctypes
    out = (ctypes.c_int64 * 2)()
    raise_for_status(N.lib().ls_query_multi_config(dtype_code(dtype), n_local, out))
    return {"grid": int(out[0]), "tile_elems": int(out[1])}


def query_cluster(dtype: torch.dtype) -> dict:
    """The latency kernel: blocks per cluster (0 = off), elements per block
    of the small and mid geometries, co-resident mid clusters, the largest n
    it takes (``max_elems``) and the largest single-cluster n
    (``one_cluster_elems``)."""
    import ctypes
    out = (ctypes.c_int64 * 6)()
    raise_for_status(N.lib().ls_query_cluster(dtype_code(dtype), out))
    return {"max_blocks": int(out[0]), "block_elems": int(out[1]), "capacity": int(out[2]),
            "max_elems": int(out[3]), "one_cluster_elems": int(out[0]) * int(out[1]),
            "mid_block_elems": int(out[4]), "mid_max_elems": int(out[5])}


class force_path:
    """Context manager pinning the kernel choice (tests / labs):
    ``"auto"``, ``"persistent"`` (never the cluster kernel) or ``"cluster"``
    (whenever n fits one cluster).  Process-wide."""

    _codes = {"auto": 0, "persistent": 1, "cluster": 2}

    def __init__(self, path: str):
        self.code = self._codes[path]

    def __enter__(self):
        raise_for_status(N.lib().ls_debug_force_path(self.code))
        return self

    def __exit__(self, *exc):
        N.lib().ls_debug_force_path(0)


def check_workspace_error(device: Optional[torch.device] = None) -> None:
    """Raise the first device-side error (liveness / protocol) recorded in the
    current stream's workspace, if any (synchronises)."""
    device = device or torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream(device)
    ws = _workspaces.get((device.index, stream.cuda_stream))
    if ws is None:
        return
    raise_for_status(N.lib().ls_workspace_error(ws.data_ptr(), ws.numel(), stream.cuda_stream))


class debug:
    """Context manager arming the device debug hooks (process-wide):

    * ``spin_budget``      look-back watchdog -> ``LivenessError`` (ChainConfig.spin_budget, chained.py:222)
    * ``corrupt_tile``     that tile publishes the identity (ChainConfig.corrupt_slot, chained.py:224)
    * ``protocol_checks``  publish-once check -> ``ProtocolViolation`` (chained.py:114-120)
    * ``reducer_delay_ns`` / ``scanner_delay_ns``  timing perturbation (test_chained.py:239-256)
    * ``stall_tile``       that tile never publishes (needs ``spin_budget``; test_chained.py:259-272)

    While armed (any of the first three), every scan synchronises and raises
    the device error word."""

    _lock = threading.Lock()

    def __init__(self, spin_budget: int = 0, corrupt_tile: int = -1, protocol_checks: bool = False,
                 reducer_delay_ns: int = 0, scanner_delay_ns: int = 0, stall_tile: int = -1):
        self.args = (spin_budget, corrupt_tile, 1 if protocol_checks else 0)
        self.perturb = (reducer_delay_ns, scanner_delay_ns, stall_tile)

    def __enter__(self):
        debug._lock.acquire()
        L = N.lib()
        raise_for_status(L.ls_debug_config(*self.args))
        raise_for_status(L.ls_debug_perturb(*self.perturb))
        return self

    def __exit__(self, *exc):
        L = N.lib()
        L.ls_debug_config(0, -1, 0)
        L.ls_debug_perturb(0, 0, -1)
        debug._lock.release()
