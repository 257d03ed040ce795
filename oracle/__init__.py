"""CPU oracle for the inclusive sum-scan path — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package, and only as
the checker (or the timed CPU baseline).  The product package
``paper_1604_04815_b200`` never imports it and has no CPU fallback.

What it restates (reference = ``chainscan`` 0.1.0, pure Python + numpy):

* ``generate_input``     bench.py:77-87   seeded full-range ints / U[-1,1] floats
* ``sequential_scan``    reference.py:61-67 -> operators.py:87-94
                         (``np.add.accumulate`` with the dtype pinned, wrapping)
* ``exclusive_scan``     derived mode, SURVEY §8a row a19
* ``float_add_envelope`` bench.py:90-92
* ``validate_output``    bench.py:95-114 (exact for ints, running envelope for
                         float add with FLOAT_EPS_REL bench.py:49)
* ``c_sequential_scan`` / ``c_chained_scan`` / ``c_reduce_sum``: the same
  algorithms in C (``lscan_oracle.c``), the chained one on real threads with
  cyclic block ownership (chained.py:264-287) — the timed CPU baseline.

Parity pin: ``tests/golden/`` holds fixtures produced by importing the real
reference in the build container (``tests/golden/make_golden.py``); the
tests check every function here against them before anything is checked
against this oracle.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from typing import Iterator, Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblscan_oracle.so")

# bench.py:36-49
FLOAT_EPS_REL = {"f32": 1e-5, "f64": 1e-12}
PAPER_NS = [32_000_000, 64_000_000, 128_000_000, 256_000_000, 512_000_000]
DEFAULT_NS = [2 ** 20, 2 ** 22, 2 ** 24, 2 ** 26]

# operators.py:24-29
DTYPES = {
    "i32": np.dtype(np.int32),
    "i64": np.dtype(np.int64),
    "f32": np.dtype(np.float32),
    "f64": np.dtype(np.float64),
}
DT_CODE = {"i32": 0, "i64": 1, "f32": 2, "f64": 3}


def tok_of(dtype) -> str:
    dtype = np.dtype(dtype)
    for tok, dt in DTYPES.items():
        if dt == dtype:
            return tok
    raise ValueError(f"no token for dtype {dtype}")


def generate_input(n: int, tok, seed) -> np.ndarray:
    """Deterministic input (bench.py:77-87): full-range ints, U[-1,1] floats."""
    dtype = DTYPES[tok] if isinstance(tok, str) else np.dtype(tok)
    rng = np.random.default_rng(seed)
    if dtype.kind == "i":
        info = np.iinfo(dtype)
        return rng.integers(info.min, info.max, size=n, dtype=dtype, endpoint=True)
    return rng.uniform(-1.0, 1.0, size=n).astype(dtype)


def generate_input_chunks(n: int, tok, seed, chunk: int) -> Iterator[np.ndarray]:
    """Stream-identical chunked ``generate_input`` (one Generator, sequential
    draws): concatenating the chunks equals ``generate_input(n, tok, seed)``.
    Used for arrays too large to hold twice in host RAM."""
    dtype = DTYPES[tok] if isinstance(tok, str) else np.dtype(tok)
    rng = np.random.default_rng(seed)
    done = 0
    while done < n:
        k = min(chunk, n - done)
        if dtype.kind == "i":
            info = np.iinfo(dtype)
            yield rng.integers(info.min, info.max, size=k, dtype=dtype, endpoint=True)
        else:
            yield rng.uniform(-1.0, 1.0, size=k).astype(dtype)
        done += k


# operators.py:111-127: ufunc and identity per operator
UFUNCS = {"add": np.add, "max": np.maximum, "min": np.minimum}


def identity(op: str, dtype) -> object:
    dtype = np.dtype(dtype)
    if op == "add":
        return dtype.type(0)
    if op == "max":
        return dtype.type(np.iinfo(dtype).min if dtype.kind == "i" else -np.inf)
    return dtype.type(np.iinfo(dtype).max if dtype.kind == "i" else np.inf)


def sequential_scan(x: np.ndarray, out: Optional[np.ndarray] = None, op: str = "add") -> np.ndarray:
    """The oracle (reference.py:61-67 / operators.py:87-94): strict left fold
    of ``op`` in the element dtype; integer overflow wraps (two's complement)."""
    x = np.asarray(x)
    if out is None:
        out = np.empty_like(x)
    if x.size == 0:
        return out
    with np.errstate(over="ignore"):
        UFUNCS[op].accumulate(x, out=out, dtype=x.dtype)
    return out


def exclusive_scan(x: np.ndarray, op: str = "add") -> np.ndarray:
    """Derived exclusive scan: y[0] = identity, y[j] = inclusive[j-1]."""
    x = np.asarray(x)
    out = np.empty_like(x)
    if x.size == 0:
        return out
    out[0] = identity(op, x.dtype)
    if x.size > 1:
        sequential_scan(x[:-1], out=out[1:], op=op)
    return out


def float_add_envelope(x: np.ndarray, eps_rel: float) -> np.ndarray:
    """Pointwise tolerance eps_rel * running sum of |x| in float64 (bench.py:90-92)."""
    return eps_rel * np.add.accumulate(np.abs(x, dtype=np.float64))


def validate_output(x: np.ndarray, y: np.ndarray, ref: Optional[np.ndarray] = None,
                    exclusive: bool = False, op: str = "add") -> Optional[str]:
    """bench.py:95-114: None if y matches the oracle, else a message.

    Integers and max/min must be bit-exact; float add must lie within
    ``FLOAT_EPS_REL * cumsum|x|`` (f32 1e-5, f64 1e-12).  For the exclusive
    mode the envelope is the inclusive one shifted by one element."""
    x = np.asarray(x)
    y = np.asarray(y)
    if ref is None:
        ref = exclusive_scan(x, op) if exclusive else sequential_scan(x, op=op)
    if y.shape != ref.shape:
        return f"shape mismatch {y.shape} vs {ref.shape}"
    if x.dtype.kind == "i" or op in ("max", "min"):
        if np.array_equal(ref, y):
            return None
        bad = np.nonzero(ref != y)[0]
        j = int(bad[0])
        return (f"validation failed at index {j}/{y.size}: "
                f"expected {ref[j]!r}, got {y[j]!r} ({bad.size} mismatches)")
    eps_rel = FLOAT_EPS_REL["f32" if x.dtype.itemsize == 4 else "f64"]
    tol = float_add_envelope(x, eps_rel)
    if exclusive and tol.size:
        tol = np.concatenate([[0.0], tol[:-1]])
    err = np.abs(y.astype(np.float64) - ref.astype(np.float64))
    bad = np.nonzero(err > tol)[0]
    if bad.size == 0:
        return None
    j = int(bad[0])
    return (f"validation failed at index {j}/{y.size}: "
            f"|{y[j]!r} - {ref[j]!r}| = {err[j]:.3e} > tol {tol[j]:.3e} "
            f"({bad.size} indices out of envelope)")


# ---------------------------------------------------------------- C oracle --

_lib = None


def build(force: bool = False) -> str:
    """Compile lscan_oracle.c (gcc, via the committed Makefile)."""
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(HERE, "lscan_oracle.c"))):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        vp, i64 = ctypes.c_void_p, ctypes.c_int64
        L.oracle_sequential_scan.argtypes = [ctypes.c_int, vp, vp, i64, ctypes.c_int, vp, vp]
        L.oracle_sequential_scan.restype = ctypes.c_int
        L.oracle_chained_scan.argtypes = [ctypes.c_int, vp, vp, i64, i64, ctypes.c_int, i64]
        L.oracle_chained_scan.restype = ctypes.c_int
        L.oracle_reduce_sum.argtypes = [ctypes.c_int, vp, i64, vp]
        L.oracle_reduce_sum.restype = ctypes.c_int
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data


def c_sequential_scan(x: np.ndarray, out: Optional[np.ndarray] = None, exclusive: bool = False,
                      carry=None) -> Tuple[np.ndarray, object]:
    """C strict left fold; returns (y, inclusive total).  ``carry`` seeds the fold."""
    x = np.ascontiguousarray(x)
    if out is None:
        out = np.empty_like(x)
    tok = tok_of(x.dtype)
    c = None if carry is None else np.array([carry], dtype=x.dtype)
    tot = np.zeros(1, dtype=x.dtype)
    rc = lib().oracle_sequential_scan(DT_CODE[tok], _ptr(x), _ptr(out), x.size,
                                      int(exclusive), _ptr(c), _ptr(tot))
    if rc:
        raise RuntimeError(f"oracle_sequential_scan rc={rc}")
    return out, tot[0]


def c_chained_scan(x: np.ndarray, out: Optional[np.ndarray] = None, block_len: int = 8192,
                   workers: Optional[int] = None, corrupt_block: int = -1) -> np.ndarray:
    """C threaded restatement of ``chained_scan`` (chained.py:316-357)."""
    x = np.ascontiguousarray(x)
    if out is None:
        out = np.empty_like(x)
    workers = workers or (os.cpu_count() or 1)
    rc = lib().oracle_chained_scan(DT_CODE[tok_of(x.dtype)], _ptr(x), _ptr(out), x.size,
                                   block_len, workers, corrupt_block)
    if rc:
        raise RuntimeError(f"oracle_chained_scan rc={rc}")
    return out


def c_reduce_sum(x: np.ndarray):
    x = np.ascontiguousarray(x)
    tot = np.zeros(1, dtype=x.dtype)
    rc = lib().oracle_reduce_sum(DT_CODE[tok_of(x.dtype)], _ptr(x), x.size, _ptr(tot))
    if rc:
        raise RuntimeError(f"oracle_reduce_sum rc={rc}")
    return tot[0]


def chunked_sequential_digest(n: int, tok: str, seed, chunk: int = 1 << 24):
    """sha256 of the oracle output for arrays too large to materialise twice:
    generates the input chunkwise and carries the fold across chunks (bit-
    identical to the one-shot fold, chained.py:290-313).  Returns
    (hexdigest, last element)."""
    import hashlib
    h = hashlib.sha256()
    carry = None
    last = None
    for xc in generate_input_chunks(n, tok, seed, chunk):
        yc, tot = c_sequential_scan(xc, carry=carry)
        h.update(yc.tobytes())
        carry = tot
        last = yc[-1]
    return h.hexdigest(), last
