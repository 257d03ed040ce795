"""The numpy drop-in ``chained_scan(problem, config)`` on the device,
replaying the shape of the reference's own chained tests
(test_chained.py, test_acceptance.py C1/C2/C6/C7) against the oracle."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1604_04815_b200 as P  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True, scope="module")
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")


def test_c1_oracle_equivalence_integers(oracle_lib):
    # test_acceptance.py:55-82 for op add: N sweep x seeds, bit-exact
    ns = (0, 1, 2, 3, 7, 8, 31, 32, 33, 1024, 100_000, 1_000_000)
    for tok in ("i32", "i64"):
        op = P.make_operator("add", tok)
        for seed in range(5):
            for n in ns:
                x = oracle_lib.generate_input(n, tok, [seed, n])
                y = P.chained_scan(P.ScanProblem(x, op))
                assert np.array_equal(y, oracle_lib.sequential_scan(x)), (tok, seed, n)


def test_c2_float_envelope(oracle_lib):
    # test_acceptance.py:85-111: N = 1e6, within eps_rel * running |x| sum
    n = 1_000_000
    for tok in ("f32", "f64"):
        op = P.make_operator("add", tok)
        x = oracle_lib.generate_input(n, tok, [7, n])
        y = P.chained_scan(P.ScanProblem(x, op))
        assert oracle_lib.validate_output(x, y) is None


def test_c7_in_place_and_returns_out(oracle_lib):
    # test_acceptance.py:246-262, test_chained.py:185-192
    op = P.make_operator("add", "i64")
    for trial in range(5):
        x = oracle_lib.generate_input(100_000, "i64", [trial, 77])
        want = P.chained_scan(P.ScanProblem(x, op))
        buf = x.copy()
        got = P.chained_scan(P.ScanProblem(buf, op, out=buf))
        assert got is buf and np.array_equal(buf, want)
    out = np.empty(1000, dtype=np.int64)
    x = oracle_lib.generate_input(1000, "i64", 1)
    assert P.chained_scan(P.ScanProblem(x, op, out=out)) is out


def test_multi_chunk_host_pipeline(oracle_lib):
    # > one 64 MiB device chunk: the carry crosses chunk launches
    n = 40_000_003
    for tok in ("i32", "f64"):
        op = P.make_operator("add", tok)
        x = oracle_lib.generate_input(n, tok, [1, n])
        y = P.chained_scan(P.ScanProblem(x, op))
        if tok == "i32":
            assert np.array_equal(y, oracle_lib.c_sequential_scan(x)[0])
        else:
            assert oracle_lib.validate_output(x, y, ref=oracle_lib.c_sequential_scan(x)[0]) is None
        ye = P.chained_exclusive_scan(P.ScanProblem(x, op))
        if tok == "i32":
            assert np.array_equal(ye, oracle_lib.c_sequential_scan(x, exclusive=True)[0])
            # in place through the pageable staging path, several chunks
            buf = x.copy()
            assert P.chained_scan(P.ScanProblem(buf, op, out=buf)) is buf
            assert np.array_equal(buf, y)


def test_pinned_host_buffers(oracle_lib):
    n = 20_000_001
    x = oracle_lib.generate_input(n, "i32", [2, n])
    xp = torch.empty(n, dtype=torch.int32).pin_memory()
    yp = torch.empty(n, dtype=torch.int32).pin_memory()
    xp.numpy()[:] = x
    y = P.chained_scan(P.ScanProblem(xp.numpy(), P.make_operator("add", "i32"), out=yp.numpy()))
    assert np.array_equal(y, oracle_lib.c_sequential_scan(x)[0])


@pytest.mark.parametrize("n", [23_068_671, 23_068_672, 30_000_017])
def test_pinned_multi_chunk(oracle_lib, n):
    # pinned (direct DMA) path over several 32 MiB chunks, ragged last chunk
    x = oracle_lib.generate_input(n, "i32", [3, n])
    xp = torch.empty(n, dtype=torch.int32).pin_memory()
    yp = torch.empty(n, dtype=torch.int32).pin_memory()
    xp.numpy()[:] = x
    y = P.chained_scan(P.ScanProblem(xp.numpy(), P.make_operator("add", "i32"), out=yp.numpy()))
    assert np.array_equal(y, oracle_lib.c_sequential_scan(x)[0])
    ye = P.chained_exclusive_scan(P.ScanProblem(xp.numpy(), P.make_operator("add", "i32"), out=yp.numpy()))
    assert np.array_equal(ye, oracle_lib.c_sequential_scan(x, exclusive=True)[0])


def test_corrupt_slot_breaks_only_downstream(oracle_lib):
    # test_chained.py:275-284 on the device: tile 1 publishes the identity
    cfg_q = P.query_config(torch.int64, 1 << 20)
    T = cfg_q["tile_elems"]
    x = np.ones(T * 4, dtype=np.int64)
    op = P.make_operator("add", "i64")
    good = P.chained_scan(P.ScanProblem(x, op))
    bad = P.chained_scan(P.ScanProblem(x, op), P.ChainConfig(corrupt_slot=1))
    assert np.array_equal(good, oracle_lib.sequential_scan(x))
    assert not np.array_equal(bad, good)
    assert np.array_equal(bad[:2 * T], good[:2 * T])


def test_spin_budget_armed_does_not_fire_on_healthy_runs(oracle_lib):
    op = P.make_operator("add", "i32")
    x = oracle_lib.generate_input(3_000_000, "i32", [1, 1])
    y = P.chained_scan(P.ScanProblem(x, op), P.ChainConfig(spin_budget=50_000_000))
    assert np.array_equal(y, oracle_lib.sequential_scan(x))


def test_c6_worker_count_is_irrelevant(oracle_lib):
    # test_acceptance.py:226-243: integer output identical for any B
    op = P.make_operator("add", "i32")
    x = oracle_lib.generate_input(100_000, "i32", [0, 61])
    outs = [P.chained_scan(P.ScanProblem(x, op), P.ChainConfig(b=b)) for b in (1, 2, 4, 8, 16)]
    for y in outs[1:]:
        assert np.array_equal(outs[0], y)


def test_on_block_hook_rejected():
    op = P.make_operator("add", "i32")
    with pytest.raises(ValueError):
        P.chained_scan(P.ScanProblem(np.ones(10, dtype=np.int32), op),
                       P.ChainConfig(on_block=lambda w, b: None))


def test_c8_throughput_over_sequential(oracle_lib):
    # test_acceptance.py:265-290 (C8): the chained scan must beat the reference's
    # sequential numpy fold by >= 1.5x at 2^26 — here through the numpy drop-in
    # with pageable host arrays (PCIe and staging included) and on the device
    import time
    n = 1 << 26
    x = oracle_lib.generate_input(n, "i32", [0, n])
    op = P.make_operator("add", "i32")
    y = P.chained_scan(P.ScanProblem(x, op))  # warm
    t0 = time.perf_counter()
    ref = oracle_lib.sequential_scan(x)
    t_seq = time.perf_counter() - t0
    t0 = time.perf_counter()
    y = P.chained_scan(P.ScanProblem(x, op))
    t_ours = time.perf_counter() - t0
    assert np.array_equal(y, ref)
    assert t_seq / t_ours >= 1.5, (t_seq, t_ours)
    xd = torch.from_numpy(x).cuda()
    yd = P.inclusive_scan(xd)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        P.inclusive_scan(xd, out=yd)
    torch.cuda.synchronize()
    t_dev = (time.perf_counter() - t0) / 10
    assert t_seq / t_dev >= 100, (t_seq, t_dev)


@pytest.mark.parametrize("tok", ["i32", "i64"])
@pytest.mark.parametrize("pinned", [True, False])
def test_host_pipeline_chunk_counts(oracle_lib, tok, pinned):
    """The host pipeline over 2-5 chunks of 32 MiB with ragged last chunks
    (sizes from an A/B of ramped head / tail chunks, which measured equal to
    equal chunks and was dropped): exact, inclusive and exclusive, pinned
    (direct DMA) and pageable (staged)."""
    es = 4 if tok == "i32" else 8
    chunk = (32 << 20) // es
    ramp = sum(chunk >> s for s in range(1, 6))
    op = P.make_operator("add", tok)
    for n in (2 * ramp + chunk, 2 * ramp + chunk + 1, 3 * chunk + 2 * ramp + 777):
        x = oracle_lib.generate_input(n, tok, [4, n])
        if pinned:
            tdt = torch.int32 if tok == "i32" else torch.int64
            xp = torch.empty(n, dtype=tdt).pin_memory()
            yp = torch.empty(n, dtype=tdt).pin_memory()
            xp.numpy()[:] = x
            xs, ys = xp.numpy(), yp.numpy()
        else:
            xs, ys = x, np.empty_like(x)
        y = P.chained_scan(P.ScanProblem(xs, op, out=ys))
        assert np.array_equal(y, oracle_lib.c_sequential_scan(x)[0]), (tok, n, pinned)
        ye = P.chained_exclusive_scan(P.ScanProblem(xs, op, out=ys))
        assert np.array_equal(ye, oracle_lib.c_sequential_scan(x, exclusive=True)[0]), (tok, n, pinned)


@pytest.mark.parametrize("threads", [8, 16])
def test_pageable_staging_copies_every_byte(threads):
    """Pageable arrays are staged with a threaded host memcpy split into
    page-rounded parts; chunks whose byte count is one element past a multiple
    of threads x 4096 once lost their last element (the parts covered
    threads x floor(bytes / threads)).  Run in a subprocess so the thread count
    (read once per process) is the one under test."""
    import os
    import subprocess
    import sys
    import textwrap
    chunk = (32 << 20) // 4
    n = 2 * chunk + threads * 1024 * 480 + 1   # last chunk: threads*4096*480 + 4 bytes
    code = textwrap.dedent(f"""
        import numpy as np, sys
        sys.path.insert(0, {os.path.dirname(os.path.dirname(os.path.abspath(__file__)))!r})
        import paper_1604_04815_b200 as P
        x = (np.arange({n}, dtype=np.int64) % 1000 - 500).astype(np.int32)
        y = P.chained_scan(P.ScanProblem(x, P.make_operator("add", "i32")))
        ref = np.cumsum(x, dtype=np.int64).astype(np.int32)
        assert np.array_equal(y, ref), int(np.nonzero(y != ref)[0][0])
        buf = x.copy()
        P.chained_scan(P.ScanProblem(buf, P.make_operator("add", "i32"), out=buf))
        assert np.array_equal(buf, ref)
        print("ok")
    """)
    env = dict(os.environ, LSCAN_HOST_COPY_THREADS=str(threads))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]
