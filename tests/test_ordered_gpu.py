"""The strict left fold on the device (``ls_ordered_scan``) and the drop-in's
``ChainConfig(b=1)`` contract: bit-identical to the sequential oracle for
float add (the reference's B = 1 path, chained.py:290-313, tested by its
test_chained.py:221-226 and test_acceptance.py:85-111), raw bits compared."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import paper_1604_04815_b200 as P  # noqa: E402
from paper_1604_04815_b200 import scan as S  # noqa: E402

pytestmark = pytest.mark.gpu

TDT = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}


@pytest.fixture(autouse=True, scope="module")
def _need_cuda():
    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a CUDA device")


def _fold(x, op="add", carry=None, exclusive=False):
    """The sequential fold with an optional carry prepended (chained.py:290-313)."""
    uf = {"add": np.add, "max": np.maximum, "min": np.minimum}[op]
    xs = x if carry is None else np.concatenate([np.array([carry], dtype=x.dtype), x])
    with np.errstate(over="ignore"):
        inc = uf.accumulate(xs, dtype=x.dtype)
    if carry is not None:
        inc = inc[1:]
    if not exclusive:
        return inc
    first = carry if carry is not None else P.make_operator(op, x.dtype).identity
    return np.concatenate([np.array([first], dtype=x.dtype), inc[:-1]])


def _bits(a):
    return a.view(np.uint32 if a.dtype.itemsize == 4 else np.uint64)


@pytest.mark.parametrize("tok", ["f32", "f64"])
@pytest.mark.parametrize("n", [1, 2, 5, 17, 1000, 4096 + 3, 100_003, 1_000_000])
@pytest.mark.parametrize("offset", [0, 1, 3])
def test_ordered_float_add_bit_exact(oracle_lib, tok, n, offset):
    x = oracle_lib.generate_input(n + offset, tok, [n, offset])
    xd = torch.from_numpy(x).cuda()[offset:]
    want = oracle_lib.sequential_scan(x[offset:])
    got = S.ordered_scan(xd).cpu().numpy()
    assert np.array_equal(_bits(got), _bits(want))
    # the parallel kernel associates differently: for float add the two differ
    # (within the envelope) on large inputs — the point of the ordered mode
    if n >= 100_000:
        par = S.inclusive_scan(xd).cpu().numpy()
        assert oracle_lib.validate_output(x[offset:], par) is None


@pytest.mark.parametrize("tok", ["i32", "i64", "f32", "f64"])
@pytest.mark.parametrize("op", ["add", "max", "min"])
def test_ordered_modes(oracle_lib, tok, op):
    n = 70_001
    x = oracle_lib.generate_input(n, tok, [3, n])
    xd = torch.from_numpy(x).cuda()
    carry = x[:1].copy()
    cd = torch.from_numpy(carry).cuda()
    for exclusive in (False, True):
        for use_carry in (False, True):
            tot = torch.empty(1, dtype=xd.dtype, device="cuda")
            got = S.ordered_scan(xd, exclusive=exclusive, carry_in=cd if use_carry else None, total_out=tot,
                                 op=op).cpu().numpy()
            want = _fold(x, op, carry[0] if use_carry else None, exclusive)
            assert np.array_equal(_bits(got), _bits(want)), (exclusive, use_carry)
            total = _fold(x, op, carry[0] if use_carry else None)[-1]
            assert _bits(tot.cpu().numpy())[0] == _bits(np.array([total]))[0]
    # in place
    buf = xd.clone()
    S.ordered_scan(buf, buf, op=op)
    assert np.array_equal(_bits(buf.cpu().numpy()), _bits(_fold(x, op)))
    # empty: total = carry, else the identity
    e = torch.empty(0, dtype=xd.dtype, device="cuda")
    tot = torch.empty(1, dtype=xd.dtype, device="cuda")
    S.ordered_scan(e, total_out=tot, op=op)
    ident = P.make_operator(op, tok).identity
    assert _bits(tot.cpu().numpy())[0] == _bits(np.array([ident], dtype=x.dtype))[0]


@pytest.mark.parametrize("tok", ["f32", "f64"])
def test_dropin_b1_float_bit_exact(oracle_lib, tok):
    # test_acceptance.py:85-111: B = 1 bit-exact, B > 1 within the envelope
    n = 1_000_000
    op = P.make_operator("add", tok)
    x = oracle_lib.generate_input(n, tok, [7, n])
    ref = oracle_lib.sequential_scan(x)
    y1 = P.chained_scan(P.ScanProblem(x, op), P.ChainConfig(b=1))
    assert np.array_equal(_bits(y1), _bits(ref))
    for b in (4, 8):
        yb = P.chained_scan(P.ScanProblem(x, op), P.ChainConfig(b=b))
        assert oracle_lib.validate_output(x, yb) is None
    # exclusive and in place keep the B = 1 bits too
    ye = P.chained_exclusive_scan(P.ScanProblem(x, op), P.ChainConfig(b=1))
    assert np.array_equal(_bits(ye[1:]), _bits(ref[:-1])) and ye[0] == 0
    buf = x.copy()
    assert P.chained_scan(P.ScanProblem(buf, op, out=buf), P.ChainConfig(b=1)) is buf
    assert np.array_equal(_bits(buf), _bits(ref))


def test_dropin_b1_across_host_chunks(oracle_lib):
    # longer than the host pipeline's device chunk (32 MiB): the fold's carry
    # crosses chunk launches and stays exact
    n = 20_000_011
    op = P.make_operator("add", "f32")
    x = oracle_lib.generate_input(n, "f32", [11, n])
    y = P.chained_scan(P.ScanProblem(x, op), P.ChainConfig(b=1))
    assert np.array_equal(_bits(y), _bits(oracle_lib.sequential_scan(x)))
