"""Golden fixtures for float max/min where the order of equal-comparing
operands decides the bits (-0.0 vs +0.0, NaN payloads), made by running the
REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_ties_golden.py

It imports ``chainscan`` read-only from /root/reference/pkg/src and records,
for inputs built here (mixes of signed zeros, negatives / positives and NaNs
of several payloads), what the reference computes with ``make_operator``
("max" / "min", operators.py:111-127) through ``sequential_scan``
(reference.py:61-67) and through its threaded ``chained_scan``
(chained.py:316-357, 4 workers, L = 16).  Written to ``ties_cases.npz``;
nothing at test time reads /root/reference.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
NAN_BITS = {"f32": np.array([0x7FC00000, 0xFFC00000, 0x7FC00123, 0xFFC0BEEF], np.uint32),
            "f64": np.array([0x7FF8000000000000, 0xFFF8000000000000, 0x7FF8000000000123,
                             0xFFF800000000BEEF], np.uint64)}


def make(kind: str, tok: str, name: str, n: int, seed: int) -> np.ndarray:
    """The same input families as tests/test_ties_gpu.py."""
    rng = np.random.default_rng([seed, n])
    dt = np.float32 if tok == "f32" else np.float64
    sign = 1.0 if name == "min" else -1.0
    if kind == "dense_zeros":
        r = rng.random(n)
        x = np.where(r < 0.3, dt(-0.0), np.where(r < 0.6, dt(0.0), (sign * rng.random(n)).astype(dt)))
    elif kind == "sparse_zeros":
        x = (sign * (rng.random(n) + 0.5)).astype(dt)
        pos = rng.choice(n, size=min(n, 4 * max(1, n // 20000)), replace=False)
        x[pos] = np.where(rng.random(pos.size) < 0.5, dt(-0.0), dt(0.0))
    else:
        x = rng.uniform(-1, 1, n).astype(dt)
        lo = int(rng.integers(0, max(1, n - 4096)))
        pos = lo + rng.choice(min(n - lo, 4096), size=min(n - lo, 6), replace=False)
        x[pos] = NAN_BITS[tok].view(dt)[rng.integers(0, 4, pos.size)]
    return x.astype(dt)


def main() -> int:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import chainscan as cs  # noqa: E402  (reference, read-only)
    from chainscan.warp import WarpGeometry

    small = WarpGeometry(w=4, k=2, warps_per_block=2)  # test_chained.py:38, L = 16
    arrays = {}
    for tok in ("f32", "f64"):
        for name in ("max", "min"):
            op = cs.make_operator(name, tok)
            for kind in ("dense_zeros", "sparse_zeros", "nans"):
                for n in (1000, 70001):
                    x = make(kind, tok, name, n, 13)
                    key = f"{name}_{tok}_{kind}_n{n}"
                    y = cs.sequential_scan(cs.ScanProblem(x, op))
                    yc = cs.chained_scan(cs.ScanProblem(x, op), cs.ChainConfig(b=4, geometry=small))
                    assert np.array_equal(y.view(np.uint8), yc.view(np.uint8)), key
                    arrays[f"x_{key}"] = x
                    arrays[f"seq_{key}"] = y
    np.savez_compressed(os.path.join(HERE, "ties_cases.npz"), **arrays)
    print(len(arrays) // 2, "cases")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
