"""Host-side logic of the multi-GPU sharded scan on CPU with
the gloo backend: shard bounds, the one-scalar all-gather, the fixed-order
carry, and reassembly — with the oracle standing in for the device compute
(the device steps themselves are covered by the -m gpu tests of
reduce_sum / carry_from_totals / inclusive_scan(carry_in=...))."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_ops():
    import oracle

    from paper_1604_04815_b200.distributed import ShardOps

    def reduce(x):
        return torch.from_numpy(np.array([oracle.c_reduce_sum(x.numpy())], dtype=x.numpy().dtype))

    def carry(totals, rank):
        t = totals.numpy()
        _, tot = oracle.c_sequential_scan(t[:rank])  # fixed left fold of the lower ranks' totals
        return torch.from_numpy(np.array([tot], dtype=t.dtype))

    def scan(x, c, exclusive, out=None):
        y, _ = oracle.c_sequential_scan(x.numpy(), exclusive=exclusive,
                                        carry=None if c is None else c.numpy()[0])
        return torch.from_numpy(y)

    return ShardOps(reduce=reduce, carry=carry, scan=scan)


def _worker(rank, world, port, n, tok, exclusive, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        from paper_1604_04815_b200.distributed import shard_bounds, sharded_scan
        x = oracle.generate_input(n, tok, [0, n])
        lo, hi = shard_bounds(n, world, rank)
        shard = torch.from_numpy(x[lo:hi].copy())
        y = sharded_scan(shard, exclusive=exclusive, ops=_oracle_ops())
        np.save(os.path.join(outdir, f"rank{rank}.npy"), y.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tok,exclusive", [(2, "i32", False), (2, "f64", True), (3, "i64", False),
                                                 (3, "i32", True), (2, "f32", False)])
def test_sharded_scan_gloo(tmp_path, world, tok, exclusive):
    import oracle
    n = 100_003
    port = _free_port()
    mp.start_processes(_worker, args=(world, port, n, tok, exclusive, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    y = np.concatenate([np.load(tmp_path / f"rank{r}.npy") for r in range(world)])
    x = oracle.generate_input(n, tok, [0, n])
    ref = oracle.exclusive_scan(x) if exclusive else oracle.sequential_scan(x)
    if tok[0] == "i":
        assert np.array_equal(y, ref)
    else:
        # the carry is folded in rank order: identical to the one-shot fold
        assert oracle.validate_output(x, y, ref=ref, exclusive=exclusive) is None


def _cyclic_worker(rank, world, port, n_local, stripe, tok, outdir):
    """Host logic of the fused block-cyclic path without a GPU:
    ``cyclic_layout`` maps this rank's share to global indices, the oracle
    scans the global array, and ``check_cyclic`` (the bench's exact self-check
    of the fused kernel) must accept the right answer and reject corruptions
    of an interior element and of a stripe head."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle

        from paper_1604_04815_b200.distributed import check_cyclic, cyclic_layout

        class Scanner:  # the attributes check_cyclic reads
            pass
        sc = Scanner()
        sc.world, sc.rank, sc.group, sc.stripe_elems = world, rank, None, stripe
        total = n_local * world
        xg = oracle.generate_input(total, tok, [5, total])
        yg = oracle.sequential_scan(xg)
        gidx = cyclic_layout(n_local, world, stripe)(rank, np.arange(n_local))
        # every global index appears exactly once over the ranks
        np.save(os.path.join(outdir, f"idx{rank}.npy"), gidx)
        x = torch.from_numpy(xg[gidx].copy())
        y = torch.from_numpy(yg[gidx].copy())
        results = [check_cyclic(sc, x, y)]
        bad = y.clone()
        bad[n_local // 2 + 1] += 1  # interior element (on every rank)
        results.append(check_cyclic(sc, x, bad))
        bad = y.clone()
        if rank == world - 1:
            bad[stripe] += 1  # head of this rank's second stripe only
        results.append(check_cyclic(sc, x, bad))
        np.save(os.path.join(outdir, f"res{rank}.npy"), np.array(results))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,tok,n_local,stripe", [(2, "i32", 10_000, 1024), (3, "i64", 9_001, 1000),
                                                      (4, "i32", 4_096, 512)])
def test_cyclic_layout_and_check_gloo(tmp_path, world, tok, n_local, stripe):
    port = _free_port()
    mp.start_processes(_cyclic_worker, args=(world, port, n_local, stripe, tok, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    idx = np.concatenate([np.load(tmp_path / f"idx{r}.npy") for r in range(world)])
    assert np.array_equal(np.sort(idx), np.arange(n_local * world))
    for r in range(world):
        ok, bad_interior, bad_head = np.load(tmp_path / f"res{r}.npy")
        assert ok and not bad_interior and not bad_head, r
