"""Generate the golden fixtures by running the REAL reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports ``chainscan`` read-only from /root/reference/pkg/src and records
what the reference itself computes:

* ``small_cases.npz``  inputs from ``chainscan.generate_input(n, tok, [seed, n])``
  (bench.py:77-87) and outputs of ``sequential_scan`` (reference.py:61-67,
  the oracle) and ``chained_scan`` (chained.py:316-357) for edge-case sizes,
  all four dtypes;
* ``digests.json``     sha256 of inputs and oracle outputs at N = 2^20 and
  2^28 for all four dtypes (the SURVEY §8c digest table), plus the derived
  exclusive-scan digest;
* ``kats.json``        known-answer tests quoted from the reference's SPEC and
  tests (test_warp.py:94-101, test_reference.py:39-42,
  test_operators.py:55-64, test_chained.py:105-116 / :275-284).

Nothing at test time reads /root/reference: the GPU box only sees these files.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

SMALL_NS = [0, 1, 2, 3, 7, 8, 31, 32, 33, 1000, 1024, 4097, 8193]
DIGEST_NS = [2 ** 20, 2 ** 28]
TOKS = ["i32", "i64", "f32", "f64"]


def sha16(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main() -> int:
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    import chainscan as cs  # noqa: E402  (reference, read-only)
    from chainscan.warp import WarpGeometry

    assert cs.__version__ == "0.1.0"
    small = WarpGeometry(w=4, k=2, warps_per_block=2)  # test_chained.py:38, L = 16

    arrays = {}
    for tok in TOKS:
        op = cs.make_operator("add", tok)
        for seed in (0, 1):
            for n in SMALL_NS:
                if seed and n > 1024:
                    continue
                x = cs.generate_input(n, tok, [seed, n])
                y = cs.sequential_scan(cs.ScanProblem(x, op))
                yc = cs.chained_scan(cs.ScanProblem(x, op),
                                     cs.ChainConfig(b=4, geometry=small))
                key = f"{tok}_s{seed}_n{n}"
                arrays[f"x_{key}"] = x
                arrays[f"seq_{key}"] = y
                arrays[f"chained_{key}"] = yc
    # max / min through the reference's oracle (test_acceptance.py:55-82 uses add and max)
    for tok in TOKS:
        for name in ("max", "min"):
            op = cs.make_operator(name, tok)
            for n in (1, 7, 33, 1000, 8193):
                x = cs.generate_input(n, tok, [5, n])
                arrays[f"x_{name}_{tok}_n{n}"] = x
                arrays[f"seq_{name}_{tok}_n{n}"] = cs.sequential_scan(cs.ScanProblem(x, op))
    # corrupt-slot red path (test_chained.py:275-284): B=2, L=16, ones(64) i64
    op = cs.make_operator("add", "i64")
    ones = np.ones(64, dtype=np.int64)
    arrays["corrupt_good"] = cs.chained_scan(cs.ScanProblem(ones, op),
                                             cs.ChainConfig(b=2, geometry=small))
    arrays["corrupt_bad"] = cs.chained_scan(cs.ScanProblem(ones, op),
                                            cs.ChainConfig(b=2, geometry=small, corrupt_slot=1))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)

    digests = {"generator": "chainscan.generate_input(n, tok, [0, n])",
               "oracle": "chainscan.sequential_scan", "numpy": np.__version__,
               "cases": []}
    for n in DIGEST_NS:
        for tok in TOKS:
            op = cs.make_operator("add", tok)
            x = cs.generate_input(n, tok, [0, n])
            y = cs.sequential_scan(cs.ScanProblem(x, op))
            ex = np.empty_like(y)
            ex[0] = 0
            ex[1:] = y[:-1]
            digests["cases"].append({
                "n": n, "dtype": tok,
                "x_sha16": sha16(x), "y_sha16": sha16(y), "excl_sha16": sha16(ex),
                "y_last": repr(y[-1].item()), "y_head": [repr(v.item()) for v in y[:4]],
                "x_head": [repr(v.item()) for v in x[:4]],
                "abs_sum_f64": float(np.abs(x, dtype=np.float64).sum()),
            })
            print(digests["cases"][-1], flush=True)
            del x, y, ex
    with open(os.path.join(HERE, "digests.json"), "w") as f:
        json.dump(digests, f, indent=1)

    # known-answer tests, each produced by the reference itself
    kats = []

    def kat(name, tok, xs, source):
        op = cs.make_operator("add", tok)
        x = np.array(xs, dtype=op.dtype)
        y = cs.sequential_scan(cs.ScanProblem(x, op))
        kats.append({"name": name, "dtype": tok, "x": [v.item() for v in x],
                     "y": [v.item() for v in y], "source": source})

    kat("spec_example", "i32", [3, 1, 7, 0, 4, 1, 6, 3], "SPEC.md:107")
    kat("one_to_eight", "i32", list(range(1, 9)), "test_warp.py:94-101")
    kat("eight_ones", "i64", [1] * 8, "test_reference.py:39-42")
    kat("i32_wrap", "i32", [2 ** 31 - 1, 1], "test_operators.py:55-64")
    kat("i64_wrap", "i64", [2 ** 63 - 1, 1], "test_operators.py:55-64")
    # slot chain KAT (test_chained.py:105-116): block reductions 10, 5, 1
    slots = cs.CommSlots(3, np.int64, np.int64(0))
    op = cs.make_operator("add", "i64")
    lefts = [int(cs.inter_block_comm(slots, i, np.int64(r), op)) for i, r in enumerate([10, 5, 1])]
    kats.append({"name": "slot_chain", "reductions": [10, 5, 1], "lefts": lefts,
                 "slots": [int(v) for v in slots.values], "source": "test_chained.py:105-116"})
    # blocks of 4 ones -> slots [4, 8, 12, 16, 20]
    slots = cs.CommSlots(5, np.int64, np.int64(0))
    for i in range(5):
        cs.inter_block_comm(slots, i, np.int64(4), op)
    kats.append({"name": "slots_of_fours", "slots": [int(v) for v in slots.values],
                 "source": "SPEC.md:284"})
    with open(os.path.join(HERE, "kats.json"), "w") as f:
        json.dump(kats, f, indent=1)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
