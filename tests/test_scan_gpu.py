"""Parity of the sm_100a scan (through the C ABI) against the oracle.

Integers: bit-exact.  Floats: within the reference envelope
FLOAT_EPS_REL * cumsum|x| (1e-5 f32, 1e-12 f64; bench.py:49, :90-114), and
bit-reproducible run to run (the round look-back fixes the association).
"""

import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

TOKS = ["i32", "i64", "f32", "f64"]
TDT = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


@pytest.fixture(scope="module", params=["auto", "persistent"])
def S(request):
    """Every case on the automatic kernel choice (small n -> the one-cluster
    latency kernel) and again with the persistent chain forced for all n."""
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    with scan.force_path(request.param):
        yield scan


@pytest.fixture(scope="module")
def S1():
    """Automatic kernel choice only: for cases whose sizes are all above the
    cluster kernel's range (both choices would run the same kernel)."""
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")
    from paper_1604_04815_b200 import scan
    return scan


def check(x, y, oracle_lib, exclusive=False, what=""):
    if x.dtype.kind == "i":
        ref = oracle_lib.c_sequential_scan(x, exclusive=exclusive)[0]
        if not np.array_equal(ref, y):
            bad = np.nonzero(ref != y)[0]
            raise AssertionError(f"{what}: {bad.size} mismatches, first at {bad[0]}: "
                                 f"want {ref[bad[0]]} got {y[bad[0]]}")
    else:
        ref = oracle_lib.c_sequential_scan(x, exclusive=exclusive)[0]
        msg = oracle_lib.validate_output(x, y, ref=ref, exclusive=exclusive)
        assert msg is None, f"{what}: {msg}"


def run(S, x, exclusive=False, **kw):
    xd = torch.from_numpy(x).cuda()
    fn = S.exclusive_scan if exclusive else S.inclusive_scan
    return fn(xd, **kw).cpu().numpy()


def test_golden_small_cases(S, golden, oracle_lib):
    arrays = golden["arrays"]
    for key in sorted(k[2:] for k in arrays if k.startswith("x_") and k.split("_")[2].startswith("s")):
        x = arrays["x_" + key]
        ref = arrays["seq_" + key]
        y = run(S, x)
        if x.dtype.kind == "i":
            assert np.array_equal(y, ref), key
        else:
            assert oracle_lib.validate_output(x, y, ref=ref) is None, key
        if x.size:
            check(x, run(S, x, exclusive=True), oracle_lib, exclusive=True, what=key)


def test_kats(S, golden):
    for k in golden["kats"]:
        if "x" in k:
            x = np.array(k["x"], dtype={"i32": np.int32, "i64": np.int64}[k["dtype"]])
            assert run(S, x).tolist() == k["y"], k["name"]


@pytest.mark.parametrize("tok", TOKS)
def test_digest_2p20(S1, golden, oracle_lib, tok):
    case = next(c for c in golden["digests"]["cases"] if c["n"] == 2 ** 20 and c["dtype"] == tok)
    n = case["n"]
    x = oracle_lib.generate_input(n, tok, [0, n])
    assert sha16(x) == case["x_sha16"]
    y = run(S1, x)
    ye = run(S1, x, exclusive=True)
    if tok[0] == "i":
        assert sha16(y) == case["y_sha16"]
        assert sha16(ye) == case["excl_sha16"]
    else:
        check(x, y, oracle_lib, what=tok)
        check(x, ye, oracle_lib, exclusive=True, what=tok)


@pytest.mark.parametrize("tok", TOKS)
def test_digest_2p28(S1, golden, oracle_lib, tok):
    # BASELINE.json configs[1]/[2]: N = 2^28, the metric's workload
    case = next(c for c in golden["digests"]["cases"] if c["n"] == 2 ** 28 and c["dtype"] == tok)
    n = case["n"]
    x = oracle_lib.generate_input(n, tok, [0, n])
    assert sha16(x) == case["x_sha16"]
    xd = torch.from_numpy(x).cuda()
    yd = S1.inclusive_scan(xd)
    y = yd.cpu().numpy()
    if tok[0] == "i":
        assert sha16(y) == case["y_sha16"]
        assert repr(y[-1].item()) == case["y_last"]
    else:
        check(x, y, oracle_lib, what=tok)
        # deterministic association: a second run is bit-identical
        y2 = S1.inclusive_scan(xd).cpu().numpy()
        assert np.array_equal(y.view(np.uint8), y2.view(np.uint8))


@pytest.mark.parametrize("tok", TOKS)
def test_sizes_around_tiles_and_rounds(S, oracle_lib, tok):
    cfg = S.query_config(TDT[tok], 1 << 30)
    T, G = cfg["tile_elems"], cfg["grid"]
    sizes = {1, 2, 3, 4, 5, 17, T - 1, T, T + 1, 2 * T + 3, G * T - 1, G * T, G * T + 1,
             3 * G * T + 12345, 7 * G * T - 5}
    for n in sorted(sizes):
        x = oracle_lib.generate_input(n, tok, [11, n])
        check(x, run(S, x), oracle_lib, what=f"{tok} n={n}")
        check(x, run(S, x, exclusive=True), oracle_lib, exclusive=True, what=f"{tok} excl n={n}")


@pytest.mark.parametrize("tok", TOKS)
def test_in_place(S1, oracle_lib, tok):
    n = 1_000_003
    x = oracle_lib.generate_input(n, tok, [7, 77])
    xd = torch.from_numpy(x).cuda()
    got = S1.inclusive_scan(xd, out=xd)
    assert got.data_ptr() == xd.data_ptr()
    check(x, xd.cpu().numpy(), oracle_lib, what="in-place")
    x2 = torch.from_numpy(x).cuda()
    S1.exclusive_scan(x2, out=x2)
    check(x, x2.cpu().numpy(), oracle_lib, exclusive=True, what="in-place exclusive")


@pytest.mark.parametrize("tok", TOKS)
def test_misaligned_generic_path(S1, oracle_lib, tok):
    # x offset by one element: not 16-byte aligned -> the generic (non-TMA) kernel
    n = 777_777
    x = oracle_lib.generate_input(n + 1, tok, [5, n])
    xd = torch.from_numpy(x).cuda()[1:]
    assert xd.data_ptr() % 16 != 0
    y = S1.inclusive_scan(xd).cpu().numpy()
    check(x[1:].copy(), y, oracle_lib, what="misaligned")


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("shift", [1, 2, 3])
def test_congruent_misalignment_split_path(S1, oracle_lib, tok, shift):
    # x and y misaligned by the same amount (a slice scanned in place, or two
    # slices at equal offsets): one TMA-kernel launch over the aligned body,
    # y's head folded into the carry in the kernel and stored by its last CTA
    es = 4 if tok in ("i32", "f32") else 8
    if (shift * es) % 16 == 0:
        pytest.skip("aligned")
    n = 3_000_011
    x = oracle_lib.generate_input(n + shift, tok, [shift, n])
    big = torch.from_numpy(x).cuda()
    xd = big[shift:]
    assert xd.data_ptr() % 16 != 0
    tot = torch.empty(1, dtype=xd.dtype, device="cuda")
    other = torch.empty(n + shift, dtype=xd.dtype, device="cuda")[shift:]
    S1.inclusive_scan(xd, out=other, total_out=tot)
    check(x[shift:].copy(), other.cpu().numpy(), oracle_lib, what="split out-of-place")
    S1.exclusive_scan(xd, out=other)
    check(x[shift:].copy(), other.cpu().numpy(), oracle_lib, exclusive=True, what="split exclusive")
    S1.inclusive_scan(xd, out=xd)
    check(x[shift:].copy(), xd.cpu().numpy(), oracle_lib, what="split in-place")
    if tok[0] == "i":
        assert tot.item() == oracle_lib.c_sequential_scan(x[shift:].copy())[1]


@pytest.mark.parametrize("tok", TOKS)
def test_carry_in_total_out(S1, oracle_lib, tok):
    n = 3_000_001
    x = oracle_lib.generate_input(n, tok, [1, 2])
    cut = 1_234_567
    xd = torch.from_numpy(x).cuda()
    t1 = torch.empty(1, dtype=xd.dtype, device="cuda")
    t2 = torch.empty(1, dtype=xd.dtype, device="cuda")
    y1 = S1.inclusive_scan(xd[:cut].clone(), total_out=t1)
    y2 = S1.inclusive_scan(xd[cut:].clone(), carry_in=t1, total_out=t2)
    y = torch.cat([y1, y2]).cpu().numpy()
    check(x, y, oracle_lib, what="carry chain")
    ref_total = oracle_lib.c_sequential_scan(x)[1]
    if tok[0] == "i":
        assert t2.item() == ref_total
    else:
        assert abs(t2.item() - ref_total) <= oracle_lib.FLOAT_EPS_REL[
            "f32" if tok == "f32" else "f64"] * np.abs(x, dtype=np.float64).sum()


@pytest.mark.parametrize("tok", TOKS)
def test_reduce_and_carry_from_totals(S, oracle_lib, tok):
    for n in (1, 3, 1000, 4_000_037):
        x = oracle_lib.generate_input(n, tok, [2, n])
        xd = torch.from_numpy(x).cuda()
        tot = S.reduce_sum(xd).item()
        ref = oracle_lib.c_sequential_scan(x)[1]
        if tok[0] == "i":
            assert tot == ref
        else:
            assert abs(tot - ref) <= 1e-5 * np.abs(x, dtype=np.float64).sum() + 1e-30
    tots = oracle_lib.generate_input(8, tok, [4, 8])
    td = torch.from_numpy(tots).cuda()
    for r in range(8):
        c = S.carry_from_totals(td, r).item()
        want = tots[:r].sum(dtype=tots.dtype) if r else 0
        if tok[0] == "i":
            with np.errstate(over="ignore"):
                want = np.add.reduce(tots[:r], dtype=tots.dtype) if r else 0
            assert c == want
        else:
            assert abs(c - float(want)) < 1e-5


def test_empty(S):
    for tok in TOKS:
        xd = torch.empty(0, dtype=TDT[tok], device="cuda")
        tot = torch.full((1,), 5, dtype=TDT[tok], device="cuda")
        assert S.inclusive_scan(xd, total_out=tot).numel() == 0
        assert tot.item() == 0


def test_float_determinism_across_calls(S1, oracle_lib):
    for tok in ("f32", "f64"):
        x = oracle_lib.generate_input(5_000_000, tok, [0, 3])
        xd = torch.from_numpy(x).cuda()
        ys = [S1.inclusive_scan(xd).cpu().numpy() for _ in range(3)]
        for y in ys[1:]:
            assert np.array_equal(ys[0].view(np.uint8), y.view(np.uint8))


def test_rejects_bad_tensors(S):
    from paper_1604_04815_b200 import ShapeError, UnsupportedOperatorError
    with pytest.raises(UnsupportedOperatorError):
        S.inclusive_scan(torch.zeros(10, dtype=torch.int16, device="cuda"))
    with pytest.raises(ShapeError):
        S.inclusive_scan(torch.zeros(2, 2, dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError):
        S.inclusive_scan(torch.zeros(10, dtype=torch.int32))
    x = torch.zeros(100, dtype=torch.int32, device="cuda")
    with pytest.raises(ShapeError):  # partial overlap
        S.inclusive_scan(x[:50], out=x[1:51])


def test_noncontiguous_input_is_made_contiguous(S, oracle_lib):
    x = oracle_lib.generate_input(20_000, "i64", [1, 9])
    xd = torch.from_numpy(x).cuda()[::2]
    y = S.inclusive_scan(xd).cpu().numpy()
    check(x[::2].copy(), y, oracle_lib, what="strided")


@pytest.mark.slow
def test_largest_size_checksum(S1, oracle_lib):
    # 2^30 i32 (4 GiB): the top of the BASELINE sweep, compared via a digest
    n = 1 << 30
    x = np.empty(n, dtype=np.int32)
    off = 0
    for part in oracle_lib.generate_input_chunks(n, "i32", [0, n], 1 << 26):
        x[off:off + part.size] = part
        off += part.size
    ref, _ = oracle_lib.c_sequential_scan(x)
    y = S1.inclusive_scan(torch.from_numpy(x).cuda()).cpu().numpy()
    assert sha16(y) == sha16(ref)


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("xoff,yoff", [(1, 0), (0, 1), (1, 2), (3, 1)])
def test_noncongruent_misalignment_shifted(S1, oracle_lib, tok, xoff, yoff):
    # x and y misaligned differently (n >= 2^20): one shifted-window launch,
    # y's head folded into the carry in the kernel
    es = 4 if tok in ("i32", "f32") else 8
    if (xoff * es) % 16 == (yoff * es) % 16:
        pytest.skip("congruent")
    n = 2_000_003
    x = oracle_lib.generate_input(n + xoff, tok, [xoff, yoff])[xoff:].copy()
    xd = torch.empty(n + 4, dtype=TDT[tok], device="cuda")[xoff:xoff + n]
    xd.copy_(torch.from_numpy(x))
    yd = torch.empty(n + 4, dtype=TDT[tok], device="cuda")[yoff:yoff + n]
    tot = torch.empty(1, dtype=TDT[tok], device="cuda")
    c = torch.from_numpy(x[:1].copy()).cuda()
    S1.inclusive_scan(xd, out=yd, total_out=tot)
    check(x, yd.cpu().numpy(), oracle_lib, what=f"{tok} inclusive x+{xoff} y+{yoff}")
    assert torch.equal(xd.cpu(), torch.from_numpy(x))  # input untouched
    S1.exclusive_scan(xd, out=yd, carry_in=c)
    xx = np.concatenate([x[:1], x]).astype(x.dtype)
    want = oracle_lib.c_sequential_scan(xx)[0][:-1]
    if tok[0] == "i":
        assert np.array_equal(yd.cpu().numpy(), want)
        assert tot.item() == oracle_lib.c_sequential_scan(x)[1]


@pytest.mark.parametrize("tok", TOKS)
@pytest.mark.parametrize("xoff", [1, 2, 3])
def test_shifted_window_kernel(S1, oracle_lib, tok, xoff):
    # x misaligned, y aligned, add: whole tiles by the shifted-window TMA kernel
    # (two aligned smem reads and a word funnel per vector), the ragged end by
    # the latency kernel with the head's total as carry
    es = 4 if tok in ("i32", "f32") else 8
    if (xoff * es) % 16 == 0:
        pytest.skip("aligned")
    T = S1.query_config(TDT[tok], 1 << 30)["tile_elems"]
    for n in (200 * T, 200 * T + 1, 201 * T - 1, 1_000_003 + 300 * T):
        x = oracle_lib.generate_input(n, tok, [xoff, n])
        xd = torch.empty(n + 4, dtype=TDT[tok], device="cuda")[xoff:xoff + n]
        xd.copy_(torch.from_numpy(x))
        yd = torch.empty(n, dtype=TDT[tok], device="cuda")
        assert xd.data_ptr() % 16 != 0 and yd.data_ptr() % 16 == 0
        tot = torch.empty(1, dtype=TDT[tok], device="cuda")
        S1.inclusive_scan(xd, out=yd, total_out=tot)
        check(x, yd.cpu().numpy(), oracle_lib, what=f"{tok} shifted n={n}")
        S1.exclusive_scan(xd, out=yd)
        check(x, yd.cpu().numpy(), oracle_lib, exclusive=True, what=f"{tok} shifted excl n={n}")
        if tok[0] == "i":
            assert tot.item() == oracle_lib.c_sequential_scan(x)[1]


def test_workspace_cache_is_bounded_across_streams(S1):
    """A caller cycling through many streams keeps at most _WS_CACHE
    workspaces alive; results stay exact on every stream, and
    release_workspaces drops them (the next call re-creates one)."""
    import paper_1604_04815_b200 as P
    x = torch.arange(1, 5001, dtype=torch.int64, device="cuda")
    ref = torch.cumsum(x, 0)
    streams = [torch.cuda.Stream() for _ in range(S1._WS_CACHE + 16)]
    for s in streams:
        with torch.cuda.stream(s):
            y = S1.inclusive_scan(x)
        s.synchronize()
        assert torch.equal(y, ref)
    assert len(S1._workspaces) <= S1._WS_CACHE
    assert P.release_workspaces() > 0
    assert len(S1._workspaces) == 0
    assert torch.equal(S1.inclusive_scan(x), ref)
