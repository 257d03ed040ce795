"""Randomised parity: hypothesis draws (dtype, operator, mode, n, x offset,
y offset, in place, carry, kernel choice) and every draw is checked against
the oracle — ints and max/min bit-exact, float add within the reference
envelope (bench.py:49, :90-114).  Sizes span every kernel's regime (one
cluster, several clusters, the persistent chain) and every alignment case
(aligned TMA path, in-kernel head + TMA or shifted-window path, generic)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
hyp = pytest.importorskip("hypothesis")
from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

pytestmark = pytest.mark.gpu

TDT = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}

SIZES = st.one_of(st.integers(1, 5000), st.integers(5000, 300_000), st.integers(300_000, 3_000_000),
                  st.sampled_from([4096, 65536, 65537, 8192 * 148, 8192 * 148 + 1, (1 << 21) + 3,
                                   # the extra-large cluster geometry's range and just past it
                                   3_500_001, 1 << 22, (1 << 22) + 1]))


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    return scan


@settings(max_examples=120, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(tok=st.sampled_from(sorted(TDT)), op=st.sampled_from(["add", "max", "min"]), excl=st.booleans(),
       n=SIZES, xoff=st.integers(0, 3), yoff=st.integers(0, 3), in_place=st.booleans(),
       carry=st.booleans(), path=st.sampled_from(["auto", "persistent", "cluster"]), seed=st.integers(0, 2**31))
def test_random_parity(S, oracle_lib, tok, op, excl, n, xoff, yoff, in_place, carry, path, seed):
    x = oracle_lib.generate_input(n + 1, tok, [seed, n])
    c0, x = x[0], x[1:].copy()
    buf = torch.empty(n + 8, dtype=TDT[tok], device="cuda")
    xd = buf[xoff:xoff + n]
    xd.copy_(torch.from_numpy(x))
    if in_place:
        yd = xd
    else:
        yd = torch.empty(n + 8, dtype=TDT[tok], device="cuda")[yoff:yoff + n]
    cd = torch.from_numpy(np.array([c0])).cuda() if carry else None
    tot = torch.empty(1, dtype=TDT[tok], device="cuda")
    fn = S.exclusive_scan if excl else S.inclusive_scan
    with S.force_path(path):
        fn(xd, out=yd, carry_in=cd, total_out=tot, op=op)
    y = yd.cpu().numpy()
    # the oracle of a carried scan is the scan of [carry, x...]
    xx = np.concatenate([[c0], x]).astype(x.dtype) if carry else x
    inc = oracle_lib.sequential_scan(xx, op=op)
    if excl:
        ref = inc[:-1] if carry else oracle_lib.exclusive_scan(x, op)
    else:
        ref = inc[1:] if carry else inc
    what = f"{tok} {op} excl={excl} n={n} xoff={xoff} yoff={yoff} inplace={in_place} carry={carry} {path}"
    if tok[0] == "i" or op != "add":
        assert np.array_equal(y, ref), what
        assert tot.cpu().numpy()[0] == inc[-1], what
    else:
        env = oracle_lib.float_add_envelope(xx, oracle_lib.FLOAT_EPS_REL[tok])
        if excl:
            env = env[:-1] if carry else np.concatenate([[0.0], env[:-1]])
        elif carry:
            env = env[1:]
        err = np.abs(y.astype(np.float64) - ref.astype(np.float64))
        assert (err <= env + 1e-30).all(), what


@settings(max_examples=16, deadline=None, derandomize=True,
          suppress_health_check=[HealthCheck.function_scoped_fixture, HealthCheck.too_slow])
@given(tok=st.sampled_from(["i32", "i64"]), op=st.sampled_from(["add", "max"]), excl=st.booleans(),
       n=st.one_of(st.integers(1, 3_000_000), st.integers(8_000_000, 30_000_000)),
       pinned=st.booleans(), seed=st.integers(0, 2**31))
def test_random_host_pipeline(oracle_lib, tok, op, excl, n, pinned, seed):
    """The numpy drop-in's host pipeline (32 MiB device chunks, pinned DMA or
    pageable staging through the threaded memcpy) at random sizes: exact."""
    import paper_1604_04815_b200 as P
    x = oracle_lib.generate_input(n, tok, [seed, n])
    if pinned:
        xp = torch.from_numpy(x).pin_memory()
        yp = torch.empty_like(xp).pin_memory()
        xs, ys = xp.numpy(), yp.numpy()
    else:
        xs, ys = x, np.empty_like(x)
    prob = P.ScanProblem(xs, P.make_operator(op, tok), out=ys)
    y = P.chained_exclusive_scan(prob) if excl else P.chained_scan(prob)
    ref = oracle_lib.exclusive_scan(x, op) if excl else oracle_lib.sequential_scan(x, op=op)
    assert np.array_equal(y, ref), (tok, op, excl, n, pinned)
