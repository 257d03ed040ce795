"""Device side of the sharded scan on one GPU: (a) G simulated ranks — the
per-shard reduce, the device carry fold and the carried scan — reassemble
to the oracle for G in 2..8; (b) the real torch.distributed path over NCCL
at world size 1."""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    return scan


@pytest.mark.parametrize("tok", ["i32", "i64", "f32", "f64"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_simulated_ranks(S, oracle_lib, tok, world):
    from paper_1604_04815_b200.distributed import shard_bounds
    n = 6_000_017
    x = oracle_lib.generate_input(n, tok, [world, n])
    xd = torch.from_numpy(x).cuda()
    shards = [xd[slice(*shard_bounds(n, world, r))].clone() for r in range(world)]
    totals = torch.cat([S.reduce_sum(sh) for sh in shards])  # the all-gathered vector
    outs = []
    for r, sh in enumerate(shards):
        carry = S.carry_from_totals(totals, r) if r else None
        outs.append(S.inclusive_scan(sh, carry_in=carry))
    y = torch.cat(outs).cpu().numpy()
    ref = oracle_lib.c_sequential_scan(x)[0]
    if tok[0] == "i":
        assert np.array_equal(y, ref)
    else:
        assert oracle_lib.validate_output(x, y, ref=ref) is None


def test_nccl_world_one(S, oracle_lib):
    import torch.distributed as dist

    from paper_1604_04815_b200.distributed import sharded_scan
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        x = oracle_lib.generate_input(3_000_001, "i64", [1, 1])
        xd = torch.from_numpy(x).cuda()
        y = sharded_scan(xd).cpu().numpy()
        assert np.array_equal(y, oracle_lib.c_sequential_scan(x)[0])
        out = torch.empty_like(xd)
        sharded_scan(xd, exclusive=True, out=out)
        assert np.array_equal(out.cpu().numpy(), oracle_lib.c_sequential_scan(x, exclusive=True)[0])
    finally:
        dist.destroy_process_group()


def test_cyclic_scan_world_one(S, oracle_lib):
    # the fused block-cyclic scanner end to end through torch.distributed
    # (NCCL, world size 1): IPC export of the exchange region, the kernel,
    # and the exact independent check
    import torch.distributed as dist

    from paper_1604_04815_b200.distributed import CyclicScan, check_cyclic
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        n = 4_000_037
        for tok, tdt in (("i32", torch.int32), ("i64", torch.int64)):
            x = oracle_lib.generate_input(n, tok, [2, 2])
            xd = torch.from_numpy(x).cuda()
            sc = CyclicScan(tdt, n)
            try:
                tot = torch.empty(1, dtype=tdt, device="cuda")
                y = sc(xd, total_out=tot)
                ref = oracle_lib.c_sequential_scan(x)
                assert np.array_equal(y.cpu().numpy(), ref[0]) and tot.item() == ref[1]
                assert check_cyclic(sc, xd, y)
                y[12345] += 1
                assert not check_cyclic(sc, xd, y)
                ye = sc(xd, exclusive=True, op="max")
                assert np.array_equal(ye.cpu().numpy(), oracle_lib.exclusive_scan(x, "max"))
            finally:
                sc.close()
    finally:
        dist.destroy_process_group()


def test_cyclic_scan_host_pipeline_world_one(S, oracle_lib):
    # CyclicScan.scan_host: chunks of whole stripes, carry chained through the
    # global totals, copies overlapped — equals the one-shot scan
    import torch.distributed as dist

    from paper_1604_04815_b200.distributed import CyclicScan
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        for tok, tdt in (("i32", torch.int32), ("f64", torch.float64)):
            sc = CyclicScan(tdt, 1)  # probe the stripe size
            stripe = sc.stripe_elems
            sc.close()
            n = 7 * stripe + 12345
            x = oracle_lib.generate_input(n, tok, [4, 4])
            sc = CyclicScan(tdt, n)
            try:
                xp = torch.from_numpy(x).pin_memory()
                yp = torch.empty_like(xp).pin_memory()
                sc.scan_host(xp, yp, stripes_per_chunk=2)
                ref = oracle_lib.c_sequential_scan(x)[0]
                if tok[0] == "i":
                    assert np.array_equal(yp.numpy(), ref)
                else:
                    assert oracle_lib.validate_output(x, yp.numpy(), ref=ref) is None
                sc.scan_host(xp, yp, exclusive=True, op="max", stripes_per_chunk=3)
                assert np.array_equal(yp.numpy(), oracle_lib.exclusive_scan(x, "max"))
            finally:
                sc.close()
    finally:
        dist.destroy_process_group()


def test_sharded_scan_host_world_one(S, oracle_lib):
    # contiguous shards end to end from pinned host memory through
    # torch.distributed (NCCL, world size 1): copy-in, reduce, all-gather,
    # carried scan, copy-out — equals the oracle
    import torch.distributed as dist

    from paper_1604_04815_b200.distributed import sharded_scan_host
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    store = dist.TCPStore("127.0.0.1", port, 1, True)
    dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        for tok in ("i32", "i64", "f64"):
            n = 5_000_011
            x = oracle_lib.generate_input(n, tok, [5, n])
            xp = torch.from_numpy(x).pin_memory()
            yp = torch.empty_like(xp).pin_memory()
            sharded_scan_host(xp, yp)
            ref = oracle_lib.c_sequential_scan(x)[0]
            if tok[0] == "i":
                assert np.array_equal(yp.numpy(), ref)
            else:
                assert oracle_lib.validate_output(x, yp.numpy(), ref=ref) is None
            if tok == "i32":
                buf = torch.empty(n + 7, dtype=xp.dtype, device="cuda")
                sharded_scan_host(xp, yp, exclusive=True, op="max", device_buf=buf)
                assert np.array_equal(yp.numpy(), oracle_lib.exclusive_scan(x, "max"))
    finally:
        dist.destroy_process_group()
