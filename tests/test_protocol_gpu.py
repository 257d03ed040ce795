"""The carry-chain protocol under stress on the device: timing perturbation
(test_chained.py:239-256 analogue), a real stall caught by the watchdog
(:259-272), fault injection (:275-284), the publish-once check (:73-82) and
epoch reuse of one workspace across many calls."""

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


def _check(x, y, oracle_lib):
    ref = oracle_lib.c_sequential_scan(x)[0]
    if x.dtype.kind == "i":
        assert np.array_equal(y, ref)
    else:
        assert oracle_lib.validate_output(x, y, ref=ref) is None


@pytest.mark.parametrize("tok", ["i32", "i64", "f32", "f64"])
@pytest.mark.parametrize("delays", [(20_000, 0), (0, 20_000), (50_000, 30_000)])
def test_timing_perturbation_keeps_results(S, oracle_lib, tok, delays):
    # the reducer lagging the scanners (or the reverse) must not change a bit
    n = 9_000_001
    x = oracle_lib.generate_input(n, tok, [3, n])
    xd = torch.from_numpy(x).cuda()
    base = S.inclusive_scan(xd).cpu().numpy()
    with S.debug(reducer_delay_ns=delays[0], scanner_delay_ns=delays[1]):
        y = S.inclusive_scan(xd).cpu().numpy()
        ye = S.exclusive_scan(xd).cpu().numpy()
    _check(x, y, oracle_lib)
    assert np.array_equal(base.view(np.uint8), y.view(np.uint8))  # same association, same bits
    assert oracle_lib.validate_output(x, ye, exclusive=True) is None


def test_real_stall_raises_liveness(S, oracle_lib):
    from paper_1604_04815_b200 import LivenessError
    x = oracle_lib.generate_input(4_000_000, "i64", [1, 2])
    xd = torch.from_numpy(x).cuda()
    with pytest.raises(LivenessError):
        with S.debug(spin_budget=20_000, stall_tile=5):
            S.inclusive_scan(xd)
    # the workspace is usable again afterwards
    y = S.inclusive_scan(xd).cpu().numpy()
    _check(x, y, oracle_lib)


def test_stall_without_budget_is_not_armed(S, oracle_lib):
    # a stall is only honoured under a watchdog: no hang, correct output
    x = oracle_lib.generate_input(2_000_000, "i32", [1, 3])
    xd = torch.from_numpy(x).cuda()
    with S.debug(stall_tile=3):
        y = S.inclusive_scan(xd).cpu().numpy()
    _check(x, y, oracle_lib)


def test_corrupt_tile_confined_downstream(S, oracle_lib):
    n = 5_000_000
    x = oracle_lib.generate_input(n, "i32", [4, 4])
    xd = torch.from_numpy(x).cuda()
    T = S.query_config(torch.int32, n)["tile_elems"]
    good = S.inclusive_scan(xd).cpu().numpy()
    with S.debug(corrupt_tile=7):
        bad = S.inclusive_scan(xd).cpu().numpy()
    assert np.array_equal(bad[:8 * T], good[:8 * T])
    assert not np.array_equal(bad[8 * T:], good[8 * T:])


def test_protocol_checks_clean_run(S, oracle_lib):
    x = oracle_lib.generate_input(3_000_000, "f64", [5, 5])
    xd = torch.from_numpy(x).cuda()
    with S.debug(protocol_checks=True):
        y = S.inclusive_scan(xd).cpu().numpy()
    _check(x, y, oracle_lib)


def test_epoch_reuse_many_calls(S, oracle_lib):
    # one workspace, hundreds of calls of varying size: tags never collide
    rng = np.random.default_rng(0)
    xs = [oracle_lib.generate_input(int(m), "i32", [9, int(m)]) for m in rng.integers(1, 3_000_000, 12)]
    xds = [torch.from_numpy(x).cuda() for x in xs]
    refs = [oracle_lib.c_sequential_scan(x)[0] for x in xs]
    for rep in range(25):
        for x, xd, ref in zip(xs, xds, refs):
            if rep % 8 == 0:
                assert np.array_equal(S.inclusive_scan(xd).cpu().numpy(), ref)
            else:
                S.inclusive_scan(xd)
    torch.cuda.synchronize()


def test_streams_are_independent(S, oracle_lib):
    # concurrent scans on two streams use two workspaces
    x1 = oracle_lib.generate_input(20_000_000, "i32", [1, 1])
    x2 = oracle_lib.generate_input(20_000_000, "i32", [2, 2])
    d1, d2 = torch.from_numpy(x1).cuda(), torch.from_numpy(x2).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        y1 = S.inclusive_scan(d1)
    with torch.cuda.stream(s2):
        y2 = S.inclusive_scan(d2)
    torch.cuda.synchronize()
    assert np.array_equal(y1.cpu().numpy(), oracle_lib.c_sequential_scan(x1)[0])
    assert np.array_equal(y2.cpu().numpy(), oracle_lib.c_sequential_scan(x2)[0])


@pytest.mark.parametrize("tok,code", [("i32", 0), ("i64", 1), ("f32", 2), ("f64", 3)])
def test_slot_handshake_stress(S, tok, code):
    # the reference's C4 (test_acceptance.py:146-196) on the device: >= 1e6
    # reads of slots being published, zero torn pairs, flags monotone
    import ctypes

    from paper_1604_04815_b200 import _native as N
    out = (ctypes.c_int64 * 3)()
    assert N.lib().ls_debug_slot_stress(code, 150_000, 32, out) == 0, N.last_detail()
    reads, torn, regress = out
    assert reads >= 1_000_000
    assert torn == 0 and regress == 0


def test_host_threads_and_streams_concurrently(S, oracle_lib):
    """Four host threads, each on its own stream, scan different arrays of every
    kernel's range (latency, multi-cluster, persistent) at the same time, and
    the numpy drop-in runs beside them: per-(device, stream) workspaces and the
    library's per-device state must keep them apart."""
    import threading

    import paper_1604_04815_b200 as P
    sizes = [5_000, 400_000, 3_000_000, 12_000_000]
    errors = []

    def work(i):
        try:
            s = torch.cuda.Stream()
            tok = ("i32", "i64", "f32", "f64")[i]
            x = oracle_lib.generate_input(sizes[i], tok, [i, 99])
            with torch.cuda.stream(s):
                xd = torch.from_numpy(x).to("cuda", non_blocking=False)
                for _ in range(5):
                    y = S.inclusive_scan(xd)
                out = y.cpu().numpy()
            msg = oracle_lib.validate_output(x, out)
            if msg:
                errors.append((tok, msg))
        except Exception as e:  # noqa: BLE001
            errors.append((i, repr(e)))

    def dropin():
        try:
            x = oracle_lib.generate_input(3_000_001, "i32", [7, 7])
            y = P.chained_scan(P.ScanProblem(x, P.make_operator("add", "i32")))
            if not np.array_equal(y, oracle_lib.sequential_scan(x)):
                errors.append(("dropin", "mismatch"))
        except Exception as e:  # noqa: BLE001
            errors.append(("dropin", repr(e)))

    threads = [threading.Thread(target=work, args=(i,)) for i in range(4)] + [threading.Thread(target=dropin)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    torch.cuda.synchronize()
    assert not errors, errors
