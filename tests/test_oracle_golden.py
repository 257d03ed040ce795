"""Pin the CPU oracle to the reference's own outputs before trusting it.

Every fixture under tests/golden/ was produced by running the real reference
package (tests/golden/make_golden.py); these tests check the numpy and C
restatements in oracle/ against them.  CPU only.
"""

import hashlib
import os

import numpy as np
import pytest

TOKS = ["i32", "i64", "f32", "f64"]
L16 = 16  # the reference tests' SMALL geometry block_len (test_chained.py:38)


def sha16(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def small_keys(golden):
    # add cases are keyed <tok>_s<seed>_n<n>; max/min cases <op>_<tok>_n<n>
    return sorted(k[2:] for k in golden["arrays"] if k.startswith("x_") and k.split("_")[2].startswith("s"))


def op_keys(golden):
    return sorted(k[2:] for k in golden["arrays"] if k.startswith("x_") and k.split("_")[1] in ("max", "min"))


def test_max_min_oracle_matches_reference(golden, oracle_lib):
    keys = op_keys(golden)
    assert len(keys) == 2 * 4 * 5
    for key in keys:
        name, tok, n = key.split("_")
        x = golden["arrays"]["x_" + key]
        assert np.array_equal(x, oracle_lib.generate_input(int(n[1:]), tok, [5, int(n[1:])]))
        ref = golden["arrays"]["seq_" + key]
        assert np.array_equal(oracle_lib.sequential_scan(x, op=name).view(np.uint8), ref.view(np.uint8)), key
        ex = oracle_lib.exclusive_scan(x, name)
        assert ex[0] == oracle_lib.identity(name, x.dtype) and np.array_equal(ex[1:], ref[:-1])


def test_generate_input_matches_reference(golden, oracle_lib):
    for key in small_keys(golden):
        tok, s, n = key.split("_")
        seed, n = int(s[1:]), int(n[1:])
        x = oracle_lib.generate_input(n, tok, [seed, n])
        ref = golden["arrays"]["x_" + key]
        assert x.dtype == ref.dtype and np.array_equal(x, ref), key


def test_sequential_numpy_and_c_match_reference_bit_exact(golden, oracle_lib):
    for key in small_keys(golden):
        x = golden["arrays"]["x_" + key]
        ref = golden["arrays"]["seq_" + key]
        assert np.array_equal(oracle_lib.sequential_scan(x), ref), key
        y, _ = oracle_lib.c_sequential_scan(x)
        # floats too: both are strict left folds in the element type
        assert np.array_equal(y.view(np.uint8), ref.view(np.uint8)), key


def test_c_chained_matches_reference_chained(golden, oracle_lib):
    # same algorithm as chained.py's vectorized mode: identical association,
    # hence identical bits even for floats, at B=4 and L=16
    for key in small_keys(golden):
        x = golden["arrays"]["x_" + key]
        ref = golden["arrays"]["chained_" + key]
        y = oracle_lib.c_chained_scan(x, block_len=L16, workers=4)
        assert np.array_equal(y.view(np.uint8), ref.view(np.uint8)), key


def test_c_chained_corrupt_slot_reproduces_reference(golden, oracle_lib):
    ones = np.ones(64, dtype=np.int64)
    good = oracle_lib.c_chained_scan(ones, block_len=L16, workers=2)
    bad = oracle_lib.c_chained_scan(ones, block_len=L16, workers=2, corrupt_block=1)
    assert np.array_equal(good, golden["arrays"]["corrupt_good"])
    assert np.array_equal(bad, golden["arrays"]["corrupt_bad"])
    assert np.array_equal(bad[:32], good[:32]) and not np.array_equal(bad, good)


@pytest.mark.parametrize("tok", TOKS)
def test_digests_2p20(golden, oracle_lib, tok):
    case = next(c for c in golden["digests"]["cases"] if c["n"] == 2 ** 20 and c["dtype"] == tok)
    n = case["n"]
    x = oracle_lib.generate_input(n, tok, [0, n])
    assert sha16(x) == case["x_sha16"]
    y, _ = oracle_lib.c_sequential_scan(x)
    assert sha16(y) == case["y_sha16"]
    assert repr(y[-1].item()) == case["y_last"]
    ex, _ = oracle_lib.c_sequential_scan(x, exclusive=True)
    assert sha16(ex) == case["excl_sha16"]
    assert sha16(oracle_lib.exclusive_scan(x)) == case["excl_sha16"]


@pytest.mark.parametrize("tok", ["i32", "f32"])
def test_digest_2p28_chunked(golden, oracle_lib, tok):
    # the chunked oracle (generate chunkwise, carry the fold) reproduces the
    # reference's one-shot 2^28 result bit for bit
    case = next(c for c in golden["digests"]["cases"] if c["n"] == 2 ** 28 and c["dtype"] == tok)
    n = case["n"]
    full, last = oracle_lib.chunked_sequential_digest(n, tok, [0, n], chunk=1 << 25)
    assert full[:16] == case["y_sha16"]
    assert repr(last.item()) == case["y_last"]


def test_chunked_generator_is_stream_identical(oracle_lib):
    for tok in TOKS:
        n = 100_003
        whole = oracle_lib.generate_input(n, tok, [3, n])
        for chunk in (999, 1000, 1 << 14):
            parts = np.concatenate(list(oracle_lib.generate_input_chunks(n, tok, [3, n], chunk)))
            assert np.array_equal(parts, whole), (tok, chunk)


def test_kats(golden, oracle_lib):
    for k in golden["kats"]:
        if "x" not in k:
            continue
        x = np.array(k["x"], dtype=oracle_lib.DTYPES[k["dtype"]])
        assert oracle_lib.sequential_scan(x).tolist() == k["y"], k["name"]
        y, _ = oracle_lib.c_sequential_scan(x)
        assert y.tolist() == k["y"], k["name"]
    chain = next(k for k in golden["kats"] if k["name"] == "slot_chain")
    assert chain["lefts"] == [0, 10, 15] and chain["slots"] == [10, 15, 16]
    fours = next(k for k in golden["kats"] if k["name"] == "slots_of_fours")
    assert fours["slots"] == [4, 8, 12, 16, 20]
    # the same chain through the C chained restatement: blocks of 4 ones
    y = oracle_lib.c_chained_scan(np.ones(20, dtype=np.int64), block_len=4, workers=3)
    assert y[3::4].tolist() == fours["slots"]


def test_integer_wrap(oracle_lib):
    for tok, top in (("i32", 2 ** 31 - 1), ("i64", 2 ** 63 - 1)):
        dt = oracle_lib.DTYPES[tok]
        x = np.array([top, 1, 1], dtype=dt)
        y, tot = oracle_lib.c_sequential_scan(x)
        assert y[1] == np.iinfo(dt).min and y[2] == np.iinfo(dt).min + 1
        assert tot == y[-1]


@pytest.mark.parametrize("b", [1, 2, 3, 8])
def test_c_chained_worker_counts(oracle_lib, b):
    for tok in TOKS:
        n = 50_001
        x = oracle_lib.generate_input(n, tok, [b, n])
        y = oracle_lib.c_chained_scan(x, block_len=1000, workers=b)
        if tok[0] == "i" or b == 1:
            assert np.array_equal(y, oracle_lib.sequential_scan(x)), (tok, b)
        else:
            assert oracle_lib.validate_output(x, y) is None, (tok, b)


def test_carry_and_total(oracle_lib):
    for tok in TOKS:
        x = oracle_lib.generate_input(10_000, tok, [9, 1])
        y_full, tot_full = oracle_lib.c_sequential_scan(x)
        y1, t1 = oracle_lib.c_sequential_scan(x[:4321])
        y2, t2 = oracle_lib.c_sequential_scan(x[4321:], carry=t1)
        assert np.array_equal(np.concatenate([y1, y2]), y_full)
        assert t2 == tot_full
        assert oracle_lib.c_reduce_sum(x[:10]) == oracle_lib.sequential_scan(x[:10])[-1]


def test_validate_output_contract(oracle_lib):
    # bench.py:95-114 behaviour (test_bench_cli.py:48-68)
    x = oracle_lib.generate_input(1000, "i64", 3)
    y = oracle_lib.sequential_scan(x)
    assert oracle_lib.validate_output(x, y) is None
    bad = y.copy()
    bad[500] += 1
    msg = oracle_lib.validate_output(x, bad)
    assert msg is not None and "500" in msg
    xf = oracle_lib.generate_input(1000, "f32", 3)
    yf = oracle_lib.sequential_scan(xf)
    assert oracle_lib.validate_output(xf, yf) is None
    jitter = yf + (np.abs(yf) * 1e-7).astype(np.float32)
    assert oracle_lib.validate_output(xf, jitter) is None
    broken = yf.copy()
    broken[10] += np.float32(1.0)
    assert oracle_lib.validate_output(xf, broken) is not None


def test_empty(oracle_lib):
    for tok in TOKS:
        x = np.empty(0, dtype=oracle_lib.DTYPES[tok])
        y, tot = oracle_lib.c_sequential_scan(x)
        assert y.size == 0 and tot == 0
        assert oracle_lib.c_chained_scan(x).size == 0


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_float_max_min_tie_semantics(oracle_lib, dt):
    """Pins the numpy behaviour the GPU operators restate (lscan_common.cuh
    float_keep_a): maximum(a, b) = (a > b || isnan(a)) ? a : b — equal operands
    give the right one, a NaN on the left beats one on the right."""
    z = np.array([-0.0, 0.0, -1.0, 0.0, -0.0], dt)
    assert np.signbit(oracle_lib.sequential_scan(z, op="max")).tolist() == [True, False, False, False, True]
    assert np.signbit(oracle_lib.sequential_scan(-z, op="min")).tolist() == [False, True, True, True, False]
    qn = np.array([np.nan], dt)
    x = np.array([1.0, -qn[0], qn[0], 3.0], dt)
    for op in ("max", "min"):
        y = oracle_lib.sequential_scan(x, op=op)
        assert not np.isnan(y[0]) and np.isnan(y[1:]).all() and np.signbit(y[1:]).all(), op


def test_ties_oracle_matches_reference(oracle_lib):
    """tests/golden/ties_cases.npz: float max/min over signed-zero mixes and NaN
    payloads, computed by the real reference (sequential_scan and its threaded
    chained_scan agree bit for bit) — the oracle restates them exactly."""
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ties_cases.npz"))
    keys = sorted(k[2:] for k in z.files if k.startswith("x_"))
    assert len(keys) == 24
    for key in keys:
        name = key.split("_")[0]
        x, ref = z["x_" + key], z["seq_" + key]
        got = oracle_lib.sequential_scan(x, op=name)
        assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), key
