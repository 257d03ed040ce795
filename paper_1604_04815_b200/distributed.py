"""Multi-GPU sharded scan: one process per GPU, one tiny carry exchange.

Not in the reference (multi-device is a non-goal there); this
is the north star's sharding:

1. rank g holds the contiguous shard x[lo_g:hi_g] in its own HBM;
2. ``reduce_sum`` gives the shard total T_g (reads N/G elements);
3. one all-gather of G scalars (G * sizeof(T) bytes over NVLink / NVSwitch);
4. carry_g = T_0 (+) ... (+) T_{g-1}, folded on the device in rank order
   (so float results are deterministic);
5. ``inclusive_scan(shard, carry_in=carry_g)``: the carry seeds round 0 of
   the single-pass kernel and is fused into its one write pass.

Per-GPU traffic is 3N/G elements (reduce + scan), the metric counts 2N.

The compute steps are injectable (``ops``) so that the host-side logic —
shard bounds, exchange, carry order — is tested on CPU with the ``gloo``
backend and an oracle compute (tests/test_distributed_gloo.py); the default
ops are the CUDA ones.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous near-equal shards: the first n % world ranks get one extra."""
    if world < 1 or not 0 <= rank < world or n < 0:
        raise ValueError(f"bad shard request n={n} world={world} rank={rank}")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    hi = lo + base + (1 if rank < extra else 0)
    return lo, hi


@dataclass
class ShardOps:
    """The three compute steps of the sharded scan."""

    reduce: Callable[[torch.Tensor], torch.Tensor]                     # shard -> [1] total
    carry: Callable[[torch.Tensor, int], torch.Tensor]                 # (totals[G], rank) -> [1]
    scan: Callable[..., torch.Tensor]  # (shard, carry, exclusive, out=None) -> scanned shard


def cuda_ops(op: str = "add") -> ShardOps:
    from . import scan as S

    def _scan(x, carry, exclusive, out=None):
        return (S.exclusive_scan if exclusive else S.inclusive_scan)(x, out, carry_in=carry, op=op)

    return ShardOps(reduce=lambda x: S.reduce(x, op=op),
                    carry=lambda t, r: S.carry_from_totals(t, r, op=op), scan=_scan)


def _gather_totals(total: torch.Tensor, world: int, group) -> torch.Tensor:
    totals = torch.empty(world, dtype=total.dtype, device=total.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(totals, total.reshape(1), group=group)
    else:
        dist.all_gather(list(totals.split(1)), total.reshape(1), group=group)
    return totals


def sharded_scan(shard: torch.Tensor, *, exclusive: bool = False, group=None,
                 ops: Optional[ShardOps] = None, out: Optional[torch.Tensor] = None,
                 op: str = "add", scan_events=None) -> torch.Tensor:
    """Scan this rank's shard as part of the global array (ranks in order).

    Every rank must call this collectively.  Returns this rank's slice of the
    global scan.  ``scan_events``: an optional (start, end) pair of CUDA
    events recorded around the carried scan on the current stream (bench.py
    times the dominant kernel inside the step with them)."""
    ops = ops or cuda_ops(op)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    totals = _gather_totals(ops.reduce(shard), world, group)
    carry = ops.carry(totals, rank) if rank > 0 else None
    if scan_events is not None:
        scan_events[0].record()
    res = ops.scan(shard, carry, exclusive) if out is None else ops.scan(shard, carry, exclusive, out=out)
    if scan_events is not None:
        scan_events[1].record()
    if out is None or res is out:
        return res
    out.copy_(res)
    return out


def sharded_scan_host(xh: torch.Tensor, yh: torch.Tensor, *, exclusive: bool = False, group=None,
                      op: str = "add", chunk_elems: int = 0,
                      device_buf: Optional[torch.Tensor] = None) -> torch.Tensor:
    """End to end from host memory for contiguous shards: this rank's shard
    ``xh`` (pinned CPU tensor) -> ``yh``.  Collective.

    The carry of a contiguous shard is known only once every lower rank has
    its whole shard on the device and reduced, so the copy-out cannot start
    before every copy-in has finished: the call is one H2D DMA of the shard,
    ``ls_reduce`` (~0.15 ms per GiB, hidden in the copy's tail), the
    all-gather of G scalars, the carried scan (~0.33 ms per GiB) and one D2H
    DMA — two PCIe transfers in sequence, each at the link's one-way rate
    (the block-cyclic ``CyclicScan.scan_host`` overlaps both directions
    instead).  ``chunk_elems`` is accepted for compatibility and unused: the
    earlier chunked form spent its time in per-chunk launches and stream
    waits, not in overlap.  The shard stays resident in HBM between the two
    transfers (``device_buf``, or a fresh allocation of the shard's size)."""
    from . import scan as S
    n = xh.numel()
    if yh.numel() != n or xh.dtype != yh.dtype or xh.dim() != 1:
        raise ValueError("xh and yh must be 1-D host tensors of the same size and dtype")
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    dev = torch.device("cuda", torch.cuda.current_device())
    d = device_buf if device_buf is not None else torch.empty(n, dtype=xh.dtype, device=dev)
    if d.numel() < n or d.dtype != xh.dtype:
        raise ValueError("device_buf must hold the shard")
    d = d[:n]
    d.copy_(xh, non_blocking=True)
    total = S.reduce(d, op=op)
    totals = _gather_totals(total, world, group)
    carry = S.carry_from_totals(totals, rank, op=op) if rank > 0 else None
    fn = S.exclusive_scan if exclusive else S.inclusive_scan
    fn(d, d, carry_in=carry, op=op)
    yh.copy_(d, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return yh


# ---------------------------------------------------------------------------
# Block-cyclic multi-GPU scan with the exchange fused into the scan kernel.

def cyclic_layout(n_local: int, world: int, stripe: int):
    """Global index of every local element for the block-cyclic layout:
    stripe k of GPU g holds global elements [(k*world + g)*stripe, ... + stripe).
    Returns a function local_index -> global_index (for tests and loaders); all
    GPUs hold the same n_local, the last stripe of each GPU may be short."""
    import numpy as np

    def to_global(rank: int, j):
        j = np.asarray(j)
        k, r = np.divmod(j, stripe)
        full_rounds = n_local // stripe
        short = n_local - full_rounds * stripe
        # rounds before the (possibly short) last one are full on every GPU
        base = np.where(k < full_rounds, (k * world + rank) * stripe,
                        full_rounds * world * stripe + rank * short)
        return base + r

    return to_global


class CyclicScan:
    """One process per GPU; every GPU scans its block-cyclic share of one
    global array in a single kernel launch, exchanging stripe aggregates with
    its peers through NVLink peer memory (include/lscan.h
    ``ls_inclusive_scan_multi``).  Construct collectively; call collectively.

    ``stripe_elems`` (= grid x tile elements) fixes the layout: GPU g's local
    stripe k is global block ``k*world + g`` (see ``cyclic_layout``)."""

    def __init__(self, dtype: torch.dtype, n_local: int, group=None, grid: int = 0):
        import ctypes

        from . import _native as N
        from . import scan as S
        from .errors import raise_for_status
        self._N, self._S, self._raise = N, S, raise_for_status
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.dtype = dtype
        self.dt = S.dtype_code(dtype)
        self.n_local = int(n_local)
        self.device = torch.device("cuda", torch.cuda.current_device())
        L = N.lib()
        cfg = S.query_multi_config(dtype, self.n_local)
        self.grid = int(grid) if grid > 0 else int(cfg["grid"])
        self.stripe_elems = self.grid * int(cfg["tile_elems"])
        meta = [None] * self.world
        dist.all_gather_object(meta, (self.n_local, self.grid, str(dtype)), group=group)
        if any(m != meta[0] for m in meta):
            raise ValueError(f"every GPU must use the same n_local, grid and dtype: {meta}")
        self.xbytes = int(L.ls_xchg_bytes(self.dt, self.world, self.n_local))
        ptr = ctypes.c_void_p()
        raise_for_status(L.ls_device_alloc(self.xbytes, ctypes.byref(ptr)))
        self.xchg = ptr.value
        raise_for_status(L.ls_workspace_init(self.xchg, self.xbytes, None))
        torch.cuda.synchronize()
        handle = ctypes.create_string_buffer(64)
        raise_for_status(L.ls_ipc_get_handle(self.xchg, handle))
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=group)
        self._opened = []
        peers = []
        err = None
        try:
            for g, h in enumerate(handles):
                if g == self.rank:
                    peers.append(self.xchg)
                    continue
                p = ctypes.c_void_p()
                raise_for_status(L.ls_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(p)))
                self._opened.append(p.value)
                peers.append(p.value)
        except Exception as e:  # noqa: BLE001 - every rank must learn about it
            err = e
        # all ranks agree before anyone can block on a peer (a rank that could
        # not map its peers must not leave the others waiting in a barrier)
        ok = torch.tensor([0 if err else 1], device=self.device)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN, group=group)
        if not ok.item():
            self.close()
            raise RuntimeError(f"peer mapping failed on some rank: {err!r}" if err else
                               "peer mapping failed on another rank")
        self.peers = torch.tensor(peers, dtype=torch.int64, device=self.device)
        # nobody may push into a peer's region before that peer zeroed it
        dist.barrier(group=group)

    def __call__(self, x: torch.Tensor, out: Optional[torch.Tensor] = None, *, op: str = "add",
                 exclusive: bool = False, carry_in: Optional[torch.Tensor] = None,
                 total_out: Optional[torch.Tensor] = None) -> torch.Tensor:
        S, N = self._S, self._N
        # a call may cover a prefix of the share (the chunks of scan_host): every
        # GPU passes the same length, a multiple of stripe_elems except at the end
        if x.numel() > self.n_local or x.dtype != self.dtype or not x.is_contiguous():
            raise ValueError("x must be a contiguous (part of the) local share this scanner was built for")
        if out is None:
            out = torch.empty_like(x)
        stream = torch.cuda.current_stream(x.device)
        L = N.lib()
        ws = S.workspace(x.device, stream, L.ls_workspace_bytes(self.dt, self.n_local))
        fn = L.ls_exclusive_scan_multi if exclusive else L.ls_inclusive_scan_multi
        rc = fn(S.op_code(op), self.dt, x.data_ptr(), out.data_ptr(), x.numel(),
                None if carry_in is None else carry_in.data_ptr(),
                None if total_out is None else total_out.data_ptr(), ws.data_ptr(), ws.numel(),
                self.rank, self.world, self.xchg, self.xbytes, self.peers.data_ptr(), self.grid,
                stream.cuda_stream)
        self._raise(rc)
        return out

    def scan_host(self, xh: torch.Tensor, yh: torch.Tensor, *, op: str = "add", exclusive: bool = False,
                  stripes_per_chunk: int = 8) -> torch.Tensor:
        """End to end from host memory: this GPU's share ``xh`` (pinned CPU
        tensor) -> ``yh``.  The share is streamed in chunks of whole stripes
        (chunk c of every GPU is one contiguous segment of the global array),
        each chunk a collective cyclic scan carrying the previous chunk's
        global total, with copy-in, scan and copy-out overlapped on three
        streams.  Collective: every GPU calls it with the same sizes."""
        n = xh.numel()
        if n != self.n_local or yh.numel() != n or xh.dtype != self.dtype or yh.dtype != self.dtype:
            raise ValueError("xh / yh must be this scanner's local share")
        chunk = max(1, stripes_per_chunk) * self.stripe_elems
        nch = (n + chunk - 1) // chunk
        nb = 3
        bufs = [torch.empty(min(chunk, n), dtype=self.dtype, device=self.device) for _ in range(min(nb, nch))]
        carry = torch.empty(2, dtype=self.dtype, device=self.device)
        s_in, s_comp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        ev_in = [torch.cuda.Event() for _ in bufs]
        ev_comp = [torch.cuda.Event() for _ in bufs]
        ev_out = [torch.cuda.Event() for _ in bufs]
        s_in.wait_stream(torch.cuda.current_stream())
        for c in range(nch):
            b = c % len(bufs)
            lo, hi = c * chunk, min(n, (c + 1) * chunk)
            d = bufs[b][:hi - lo]
            if c >= len(bufs):
                s_in.wait_event(ev_out[b])
            with torch.cuda.stream(s_in):
                d.copy_(xh[lo:hi], non_blocking=True)
                ev_in[b].record(s_in)
            s_comp.wait_event(ev_in[b])
            with torch.cuda.stream(s_comp):
                self(d, d, op=op, exclusive=exclusive, carry_in=carry[(c - 1) % 2:(c - 1) % 2 + 1] if c else None,
                     total_out=carry[c % 2:c % 2 + 1])
                ev_comp[b].record(s_comp)
            s_out.wait_event(ev_comp[b])
            with torch.cuda.stream(s_out):
                yh[lo:hi].copy_(d, non_blocking=True)
                ev_out[b].record(s_out)
        s_out.synchronize()
        return yh

    def close(self):
        L = self._N.lib()
        torch.cuda.synchronize()
        for p in getattr(self, "_opened", []):
            L.ls_ipc_close(p)
        self._opened = []
        if getattr(self, "xchg", None):
            L.ls_device_free(self.xchg)
            self.xchg = None


def check_cyclic(scanner: "CyclicScan", x: torch.Tensor, y: torch.Tensor) -> bool:
    """Independent exact check of a block-cyclic integer add scan, with no
    scan of the data: within every stripe y[j] - y[j-1] == x[j] (wrapping),
    and the first element of stripe (k, g) equals the wrapped sum of every
    earlier stripe of every GPU (stripe sums all-gathered, tiny) plus x.
    Integer dtypes only."""
    if x.dtype.is_floating_point:
        raise ValueError("check_cyclic is exact and needs an integer dtype")
    n, S = x.numel(), scanner.stripe_elems
    starts = torch.arange(0, n, S, device=x.device)
    d = torch.empty_like(y)
    d[1:] = y[1:] - y[:-1]
    d[starts] = x[starts]  # stripe heads are checked against the global prefix below
    ok = bool(torch.equal(d, x))
    # stripe sums (wrapping, in the element type) of this GPU, then everyone's
    full = n // S
    parts = [x[:full * S].view(full, S).sum(1, dtype=torch.int64)]
    if n % S:
        parts.append(x[full * S:].sum(dtype=torch.int64).reshape(1))
    sums = torch.cat(parts).to(x.dtype)
    allsums = torch.empty(scanner.world, sums.numel(), dtype=x.dtype, device=x.device)
    dist.all_gather_into_tensor(allsums, sums.contiguous(), group=scanner.group) \
        if dist.get_backend(scanner.group) == "nccl" else \
        dist.all_gather(list(allsums.unbind(0)), sums, group=scanner.group)
    order = allsums.t().reshape(-1)  # global stripe order: round-major, then GPU
    excl = torch.cumsum(order.to(torch.int64), 0) - order.to(torch.int64)
    mine = excl.reshape(-1, scanner.world)[:, scanner.rank].to(x.dtype)  # wraps back to the element type
    heads = (mine + x[starts]).to(x.dtype)
    ok = ok and bool(torch.equal(y[starts], heads))
    flag = torch.tensor([1 if ok else 0], device=x.device)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=scanner.group)
    return bool(flag.item())
