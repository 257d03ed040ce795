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


def sharded_scan(shard: torch.Tensor, *, exclusive: bool = False, group=None,
                 ops: Optional[ShardOps] = None, out: Optional[torch.Tensor] = None,
                 op: str = "add") -> torch.Tensor:
    """Scan this rank's shard as part of the global array (ranks in order).

    Every rank must call this collectively.  Returns this rank's slice of the
    global scan."""
    ops = ops or cuda_ops(op)
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    total = ops.reduce(shard).reshape(1)
    totals = torch.empty(world, dtype=shard.dtype, device=shard.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(totals, total, group=group)
    else:
        parts = list(totals.split(1))
        dist.all_gather(parts, total, group=group)
    carry = ops.carry(totals, rank) if rank > 0 else None
    if out is None:
        return ops.scan(shard, carry, exclusive)
    res = ops.scan(shard, carry, exclusive, out=out)
    if res is not out:
        out.copy_(res)
    return out
