"""max / min operators on the device (operators.py:111-127):
bit-exact against the reference's outputs and the oracle for every dtype,
both scan modes, both kernel paths, the reduction and the carry fold."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOKS = ["i32", "i64", "f32", "f64"]


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    return scan


def bits_equal(a, b):
    return a.dtype == b.dtype and np.array_equal(np.ascontiguousarray(a).view(np.uint8),
                                                 np.ascontiguousarray(b).view(np.uint8))


def test_golden_max_min(S, golden):
    arrays = golden["arrays"]
    keys = sorted(k[2:] for k in arrays if k.startswith("x_") and k.split("_")[1] in ("max", "min"))
    assert keys
    for key in keys:
        name = key.split("_")[0]
        x = arrays["x_" + key]
        y = S.inclusive_scan(torch.from_numpy(x).cuda(), op=name).cpu().numpy()
        assert bits_equal(y, arrays["seq_" + key]), key


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("name", ["max", "min"])
def test_sizes_modes_paths(S, oracle_lib, tok, name):
    T = S.query_config({"i32": torch.int32, "i64": torch.int64, "f32": torch.float32,
                        "f64": torch.float64}[tok], 1 << 30)["tile_elems"]
    for n in (1, 5, T - 1, T + 3, 3_000_017):
        x = oracle_lib.generate_input(n + 1, tok, [8, n])
        xd = torch.from_numpy(x).cuda()
        for sl, xs in ((slice(0, n), x[:n]), (slice(1, n + 1), x[1:])):  # aligned / misaligned
            d = xd[sl]
            assert bits_equal(S.inclusive_scan(d, op=name).cpu().numpy(), oracle_lib.sequential_scan(xs, op=name))
            assert bits_equal(S.exclusive_scan(d, op=name).cpu().numpy(), oracle_lib.exclusive_scan(xs, name))


@pytest.mark.parametrize("tok", TOKS)
def test_reduce_carry_and_chunked_carry(S, oracle_lib, tok):
    for name in ("max", "min"):
        x = oracle_lib.generate_input(2_500_001, tok, [3, 3])
        xd = torch.from_numpy(x).cuda()
        want = oracle_lib.UFUNCS[name].reduce(x)
        assert bits_equal(S.reduce(xd, op=name).cpu().numpy(), np.array([want], dtype=x.dtype))
        # two chunks chained through carry_in / total_out
        cut = 1_000_003
        t1 = torch.empty(1, dtype=xd.dtype, device="cuda")
        y1 = S.inclusive_scan(xd[:cut].clone(), total_out=t1, op=name)
        y2 = S.inclusive_scan(xd[cut:].clone(), carry_in=t1, op=name)
        assert bits_equal(torch.cat([y1, y2]).cpu().numpy(), oracle_lib.sequential_scan(x, op=name))
        tots = torch.from_numpy(x[:8].copy()).cuda()
        for r in range(8):
            c = S.carry_from_totals(tots, r, op=name).cpu().numpy()[0]
            expect = oracle_lib.UFUNCS[name].reduce(x[:r]) if r else oracle_lib.identity(name, x.dtype)
            assert c == expect
        e = torch.empty(0, dtype=xd.dtype, device="cuda")
        assert S.reduce(e, op=name).item() == oracle_lib.identity(name, x.dtype)


def test_nan_propagates_like_numpy(S, oracle_lib):
    for tok in ("f32", "f64"):
        x = oracle_lib.generate_input(100_000, tok, [1, 1])
        x[12_345] = np.nan
        for name in ("max", "min"):
            y = S.inclusive_scan(torch.from_numpy(x).cuda(), op=name).cpu().numpy()
            ref = oracle_lib.sequential_scan(x, op=name)
            assert np.array_equal(np.isnan(y), np.isnan(ref))
            assert np.array_equal(y[~np.isnan(y)], ref[~np.isnan(ref)])


def test_dropin_c1_max(oracle_lib):
    # test_acceptance.py:55-82 runs every algorithm with add AND max: the
    # device drop-in with op max, i32/i64, bit-exact
    import paper_1604_04815_b200 as P
    for tok in ("i32", "i64"):
        op = P.make_operator("max", tok)
        for seed in range(3):
            for n in (0, 1, 2, 3, 7, 8, 31, 32, 33, 1024, 100_000, 1_000_000):
                x = oracle_lib.generate_input(n, tok, [seed, n])
                y = P.chained_scan(P.ScanProblem(x, op))
                assert np.array_equal(y, oracle_lib.sequential_scan(x, op="max")), (tok, seed, n)
    op = P.make_operator("min", "f64")
    x = oracle_lib.generate_input(50_000_003, "f64", [0, 1])
    assert bits_equal(P.chained_scan(P.ScanProblem(x, op)), oracle_lib.sequential_scan(x, op="min"))


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("name", ["add", "max", "min"])
def test_reduce_misaligned_slices(S, oracle_lib, tok, name):
    """ls_reduce over slices at every element offset (the reduction's
    16-byte head, vector body and ragged tail), sizes from one element to
    several grid strides; ints and max/min exact, float add in the envelope."""
    dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}[tok]
    for n in (1, 3, 17, 1000, 65_537, 3_000_001):
        base = oracle_lib.generate_input(n + 4, tok, [11, n])
        xd = torch.from_numpy(base).cuda()
        for off in range(4):
            x = base[off:off + n]
            got = S.reduce(xd[off:off + n], op=name).cpu().numpy().reshape(-1)[0]
            if tok[0] == "i" or name != "add":
                want = oracle_lib.sequential_scan(x, op=name)[-1]
                assert bits_equal(np.array([got]), np.array([want])), (n, off)
            else:
                want = np.add.reduce(x.astype(np.float64))
                env = oracle_lib.FLOAT_EPS_REL[tok] * np.abs(x.astype(np.float64)).sum() * 4 + 1e-30
                assert abs(float(got) - want) <= env, (n, off, got, want)
