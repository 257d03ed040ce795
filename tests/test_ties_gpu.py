"""Float max/min bit-exactness where the ORDER of equal-comparing operands
matters: numpy's maximum(a, b) = (a > b || isnan(a)) ? a : b, so the
sequential fold (the oracle, reference.py:61-67 with operators.py:87-94's
ufunc table) returns the rightmost of equal maximal elements (-0.0 vs +0.0)
and the leftmost NaN (its payload and sign).  Every path that combines
partial results out of sequence order (tile reducers, look-backs, the
reduction kernel) must still produce those bits.  Compared as raw bits."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TDT = {"f32": torch.float32, "f64": torch.float64}
NPT = {"f32": np.float32, "f64": np.float64}
UI = {"f32": np.uint32, "f64": np.uint64}


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    return scan


def nans(tok):
    """NaNs with distinct bits: +qNaN, -qNaN and two payloads."""
    if tok == "f32":
        b = np.array([0x7FC00000, 0xFFC00000, 0x7FC00123, 0xFFC0BEEF], np.uint32)
    else:
        b = np.array([0x7FF8000000000000, 0xFFF8000000000000, 0x7FF8000000000123, 0xFFF800000000BEEF], np.uint64)
    return b.view(NPT[tok])


def make(kind, tok, op, n, seed):
    rng = np.random.default_rng([seed, n])
    dt = NPT[tok]
    sign = 1.0 if op == "min" else -1.0  # max: values <= 0, min: values >= 0
    if kind == "dense_zeros":      # the running result is a zero almost everywhere
        r = rng.random(n)
        x = np.where(r < 0.3, dt(-0.0), np.where(r < 0.6, dt(0.0), (sign * rng.random(n)).astype(dt)))
    elif kind == "sparse_zeros":   # most tiles hold no zero; a few hold both signs
        x = (sign * (rng.random(n) + 0.5)).astype(dt)
        k = max(1, n // 20000)
        pos = rng.choice(n, size=min(n, 4 * k), replace=False)
        x[pos] = np.where(rng.random(pos.size) < 0.5, dt(-0.0), dt(0.0))
    elif kind == "extremes":       # infinities, magnitudes >= 2^1017 (f64) / near FLT_MAX and zeros
        x = rng.uniform(-1, 1, n).astype(dt)   # in a few tiles: the reducers' NaN screen flags
        big = np.array([np.inf, -np.inf, 2.0 ** 1020, -(2.0 ** 1020), 2.0 ** 1017, 0.0, -0.0]
                       if tok == "f64" else [np.inf, -np.inf, 3.0e38, -3.0e38, 0.0, -0.0])
        k = max(1, n // 50000)
        pos = rng.choice(n, size=min(n, 3 * k), replace=False)
        x[pos] = big[rng.integers(0, big.size, pos.size)].astype(dt)
    else:                          # "nans": several NaN payloads clustered in one region
        x = rng.uniform(-1, 1, n).astype(dt)
        lo = rng.integers(0, max(1, n - 4096))
        pos = lo + rng.choice(min(n - lo, 4096), size=min(n - lo, 6), replace=False)
        x[pos] = nans(tok)[rng.integers(0, 4, pos.size)]
    return x.astype(dt)


def seq(x, op):
    f = np.maximum if op == "max" else np.minimum
    return f.accumulate(x)


@pytest.mark.parametrize("tok", ["f32", "f64"])
@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("kind", ["dense_zeros", "sparse_zeros", "nans", "extremes"])
@pytest.mark.parametrize("n,path", [(3000, "auto"), (300_000, "auto"), (300_000, "cluster"),
                                    ((1 << 22) + 5, "persistent"), ((1 << 22) + 5, "auto")])
@pytest.mark.parametrize("excl", [False, True])
def test_ties_scan(S, tok, op, kind, n, path, excl):
    x = make(kind, tok, op, n, 7)
    xd = torch.from_numpy(x).cuda()
    tot = torch.empty(1, dtype=TDT[tok], device="cuda")
    fn = S.exclusive_scan if excl else S.inclusive_scan
    with S.force_path(path):
        y = fn(xd, total_out=tot, op=op).cpu().numpy()
    inc = seq(x, op)
    ref = np.concatenate([[-np.inf if op == "max" else np.inf], inc[:-1]]).astype(x.dtype) if excl else inc
    bad = np.flatnonzero(y.view(UI[tok]) != ref.view(UI[tok]))
    assert bad.size == 0, f"{bad.size} mismatching bits, first at {bad[:5]}"
    assert tot.cpu().numpy().view(UI[tok])[0] == inc[-1:].view(UI[tok])[0]


@pytest.mark.parametrize("tok", ["f32", "f64"])
@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("kind", ["dense_zeros", "sparse_zeros", "nans"])
def test_ties_scan_carry(S, tok, op, kind):
    n = (1 << 21) + 3
    x = make(kind, tok, op, n + 1, 11)
    c0, x = x[:1].copy(), x[1:].copy()
    y = S.inclusive_scan(torch.from_numpy(x).cuda(), carry_in=torch.from_numpy(c0).cuda(), op=op).cpu().numpy()
    ref = seq(np.concatenate([c0, x]), op)[1:]
    assert np.array_equal(y.view(UI[tok]), ref.view(UI[tok]))


@pytest.mark.parametrize("tok", ["f32", "f64"])
@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("kind", ["dense_zeros", "sparse_zeros", "nans"])
@pytest.mark.parametrize("n", [1000, 1 << 20, (1 << 24) + 7])
def test_ties_reduce(S, tok, op, kind, n):
    x = make(kind, tok, op, n, 3)
    got = S.reduce(torch.from_numpy(x).cuda(), op=op).cpu().numpy().reshape(-1)
    want = seq(x, op)[-1:]
    assert got.view(UI[tok])[0] == want.view(UI[tok])[0], (got, want)


@pytest.mark.parametrize("tok", ["f32", "f64"])
@pytest.mark.parametrize("op", ["max", "min"])
@pytest.mark.parametrize("kind", ["dense_zeros", "sparse_zeros", "nans", "extremes"])
@pytest.mark.parametrize("xoff,yoff", [(1, 0), (0, 1), (3, 2)])
def test_ties_misaligned(S, tok, op, kind, xoff, yoff):
    """x and y misaligned differently: one launch — y's head folded into the
    carry in the kernel, x through shifted TMA windows, the ragged end bounded."""
    n = (1 << 21) + 5
    x = make(kind, tok, op, n, 5)
    xb = torch.empty(n + 4, dtype=TDT[tok], device="cuda")
    xd = xb[xoff:xoff + n]
    xd.copy_(torch.from_numpy(x))
    yd = torch.empty(n + 4, dtype=TDT[tok], device="cuda")[yoff:yoff + n]
    tot = torch.empty(1, dtype=TDT[tok], device="cuda")
    S.inclusive_scan(xd, out=yd, total_out=tot, op=op)
    ref = seq(x, op)
    assert np.array_equal(yd.cpu().numpy().view(UI[tok]), ref.view(UI[tok]))
    assert tot.cpu().numpy().view(UI[tok])[0] == ref[-1:].view(UI[tok])[0]


@pytest.fixture(scope="module")
def ties_golden():
    import os
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "ties_cases.npz"))


@pytest.mark.parametrize("path", ["auto", "persistent"])
@pytest.mark.parametrize("excl", [False, True])
def test_ties_match_reference_fixtures(S, ties_golden, path, excl):
    """The CUDA scan against the reference's own outputs (tests/golden/
    make_ties_golden.py), bit for bit, on the latency and persistent kernels."""
    keys = sorted(k[2:] for k in ties_golden.files if k.startswith("x_"))
    for key in keys:
        name, tok = key.split("_")[0], key.split("_")[1]
        x, ref = ties_golden["x_" + key], ties_golden["seq_" + key]
        fn = S.exclusive_scan if excl else S.inclusive_scan
        with S.force_path(path):
            y = fn(torch.from_numpy(x).cuda(), op=name).cpu().numpy()
        if excl:
            ref = np.concatenate([[-np.inf if name == "max" else np.inf], ref[:-1]]).astype(x.dtype)
        assert np.array_equal(y.view(UI[tok]), ref.view(UI[tok])), (key, path, excl)
