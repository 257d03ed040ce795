"""``python -m paper_1604_04815_b200`` — the reference's benchmark front end
(chainscan/cli.py:39-95, :149-195) for the device scan.

    python -m paper_1604_04815_b200 --algo chained --dtype i32 --op add --n 268435456 --runs 5

Same flags, record schema, validation policy and exit codes as ``chainscan``:
0 success, 1 validation or liveness failure, 2 usage error, 3 output I/O
error.  ``--algo`` accepts ``chained`` (the device scan); the reference's CPU
algorithms and the ``simulate`` subcommand are out of scope and are usage
errors.  Timing defaults to the reference's: wall clock around one
``chained_scan(ScanProblem(numpy x))`` call (host arrays, so PCIe included),
best of ``--runs``; ``--timing device`` times the kernel alone on a
device-resident array with CUDA events.  ``--inject-slot-fault TILE`` makes
that tile publish the identity (ChainConfig.corrupt_slot), so validation
fails and the exit code is 1 — the reference's hidden flag (cli.py:79-80).
Validation follows the reference's rule on the host after timing
(records.host_check: the numpy sequential fold, raw-bit comparison for
integers and max/min, the envelope for float add).  The reference's
block-geometry flags (``--warp-width``, ``--k``, ``--warps-per-block``,
``--block-scan-mode``) are accepted and validated like the reference's
(WarpGeometry, warp.py:42-82); the device's tile shape is fixed at compile
time, so they do not change the kernel.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from typing import List, Optional

import numpy as np

from . import __version__
from .chained import ChainConfig, chained_exclusive_scan, chained_scan
from .errors import LivenessError, ProtocolViolation
from .operators import DTYPES, OPERATOR_NAMES, make_operator
from .problem import ScanProblem, ShapeError
from .records import BenchRecord, host_check, write_records

DEFAULT_NS = [2 ** 20, 2 ** 22, 2 ** 24, 2 ** 26]                                 # bench.py:47
PAPER_NS = [32_000_000, 64_000_000, 128_000_000, 256_000_000, 512_000_000]        # bench.py:45
ALGORITHMS = ("chained",)
REFERENCE_ALGORITHMS = ("sequential", "hillis-steele", "blelloch", "matrix", "chained")  # bench.py:36
WORKERS_ENV = "CHAINSCAN_WORKERS"  # cli.py:36


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(
        prog="lscan",
        description="B200 single-pass scan benchmarks (chainscan-compatible). The reference's CPU algorithms "
                    "and its `simulate` subcommand (the scheduler model) are not provided.")
    p.add_argument("--version", action="version", version=f"lscan {__version__}")
    p.add_argument("--algo", choices=REFERENCE_ALGORITHMS, default="chained",
                   help="scan algorithm (only 'chained' runs on the device; the others are usage errors)")
    p.add_argument("--dtype", choices=sorted(DTYPES), default="i32")
    p.add_argument("--op", choices=OPERATOR_NAMES, default="add")
    p.add_argument("--n", action="append", type=int, metavar="N", help="input length; repeatable")
    p.add_argument("--n-preset", choices=["paper"], help="the published sizes (32M..512M)")
    p.add_argument("--workers", type=int, default=None, help="accepted for compatibility (grid = resident CTAs)")
    p.add_argument("--warp-width", type=int, default=32, metavar="W",
                   help="accepted for compatibility: power of two in [2, 64] (the device warp is 32)")
    p.add_argument("--k", type=int, default=8, metavar="K", help="accepted for compatibility (>= 1)")
    p.add_argument("--warps-per-block", type=int, default=32, metavar="WPB",
                   help="accepted for compatibility (at most W)")
    p.add_argument("--block-scan-mode", choices=["vectorized", "warp-model"], default="vectorized",
                   help="accepted for compatibility")
    p.add_argument("--runs", type=int, default=3)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--in-place", action="store_true")
    p.add_argument("--exclusive", action="store_true", help="exclusive scan (derived mode)")
    p.add_argument("--no-validate", action="store_true")
    p.add_argument("--output", metavar="PATH")
    p.add_argument("--format", choices=["csv", "json"], default="csv")
    p.add_argument("--extended", action="store_true", help="append device/roofline columns")
    p.add_argument("--timing", choices=["host", "device"], default="host")
    p.add_argument("--inject-slot-fault", type=int, default=None, metavar="TILE", help=argparse.SUPPRESS)
    p.add_argument("command", nargs="?", help=argparse.SUPPRESS)
    return p


def _usage(msg: str) -> int:
    print(f"lscan: error: {msg}", file=sys.stderr)
    return 2


def generate_input(n: int, tok: str, seed) -> np.ndarray:
    """The reference's input recipe (bench.py:77-87)."""
    dtype = DTYPES[tok]
    rng = np.random.default_rng(seed)
    if dtype.kind == "i":
        info = np.iinfo(dtype)
        return rng.integers(info.min, info.max, size=n, dtype=dtype, endpoint=True)
    return rng.uniform(-1.0, 1.0, size=n).astype(dtype)


def _peak_gbs() -> Optional[float]:
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(here, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:
        return None


def bench_one(args, n: int) -> BenchRecord:
    import torch

    from . import scan as S
    op = make_operator(args.op, args.dtype)
    x = generate_input(n, args.dtype, [args.seed, n])
    cfg = ChainConfig(corrupt_slot=args.inject_slot_fault) if args.inject_slot_fault is not None else None
    fn = chained_exclusive_scan if args.exclusive else chained_scan
    times = []
    y = None
    if args.timing == "host":
        for _ in range(args.runs):
            if args.in_place:
                work = x.copy()
                prob = ScanProblem(work, op, out=work)
            else:
                prob = ScanProblem(x, op)
            t0 = time.perf_counter()
            y = fn(prob, cfg)
            times.append(time.perf_counter() - t0)
    else:
        xd = torch.from_numpy(x).cuda()
        yd = xd.clone() if args.in_place else torch.empty_like(xd)
        dfn = S.exclusive_scan if args.exclusive else S.inclusive_scan
        ctx = S.debug(corrupt_tile=args.inject_slot_fault) if args.inject_slot_fault is not None else None
        for _ in range(args.runs):
            src = yd if args.in_place else xd
            if args.in_place:
                yd.copy_(xd)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if ctx:
                ctx.__enter__()
            try:
                e0.record()
                dfn(src, yd, op=args.op)
                e1.record()
                torch.cuda.synchronize()
            finally:
                if ctx:
                    ctx.__exit__(None, None, None)
            times.append(e0.elapsed_time(e1) * 1e-3)
    failure = None
    verdict = "skipped"
    if not args.no_validate:
        yh = y if args.timing == "host" else yd.cpu().numpy()
        failure = host_check(x, yh, args.op, args.exclusive)
        verdict = "false" if failure else "true"
    best = min(times)
    es = x.dtype.itemsize
    peak = _peak_gbs()
    gbs = 2 * n * es / best / 1e9 if best > 0 else 0.0
    cfgq = S.query_config({"i32": torch.int32, "i64": torch.int64, "f32": torch.float32,
                           "f64": torch.float64}[args.dtype], max(n, 1))
    rec = BenchRecord(
        algorithm=args.algo, dtype=args.dtype, op=args.op, n=n, workers=cfgq["grid"],
        warp_width=32, k=cfgq["tile_elems"] // cfgq["threads"] if cfgq["threads"] else 0,
        warps_per_block=cfgq["threads"] // 32, runs=args.runs, best_seconds=best,
        mean_seconds=sum(times) / len(times), geps=(n / best) * 1e-9 if best > 0 else 0.0,
        validated=verdict, in_place="true" if args.in_place else "false", failure=failure,
        extra={"device": torch.cuda.get_device_name(), "timing": args.timing, "bytes_moved": 2 * n * es,
               "gbs": round(gbs, 1), "roofline_frac": round(gbs / peak, 4) if peak else None,
               "roofline_denominator_gbs": peak, "impl": "lscan-b200"})
    return rec


def main(argv: Optional[List[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    if args.command is not None:
        return _usage(f"subcommand {args.command!r} is not provided (only the benchmark mode is)")
    if args.algo not in ALGORITHMS:
        return _usage(f"algorithm {args.algo!r} has no device implementation; choose from {ALGORITHMS}")
    workers = args.workers
    if workers is None and os.environ.get(WORKERS_ENV):
        # cli.py:99-110: the flag wins, then the environment (validated, but
        # the device's CTA count is what runs)
        try:
            workers = int(os.environ[WORKERS_ENV])
        except ValueError:
            return _usage(f"${WORKERS_ENV} must be an integer, got {os.environ[WORKERS_ENV]!r}")
    if workers is not None and workers < 1:
        return _usage(f"--workers must be >= 1, got {workers}")
    if args.runs < 1:
        return _usage(f"--runs must be >= 1, got {args.runs}")
    # WarpGeometry's checks (warp.py:42-82)
    w = args.warp_width
    if w < 2 or w > 64 or w & (w - 1):
        return _usage(f"warp width must be a power of two in [2, 64], got {w}")
    if args.k < 1:
        return _usage(f"registers per lane must be >= 1, got {args.k}")
    if args.warps_per_block < 1 or args.warps_per_block > w:
        return _usage(f"warps_per_block must be in [1, {w}], got {args.warps_per_block}")
    ns = list(args.n) if args.n else []
    if args.n_preset == "paper":
        ns += PAPER_NS
    if not ns:
        ns = list(DEFAULT_NS)
    if any(n < 0 for n in ns):
        return _usage("--n must be >= 0")
    try:
        records = [bench_one(args, n) for n in ns]
    except (LivenessError, ProtocolViolation) as exc:
        print(f"lscan: {exc}", file=sys.stderr)
        return 1
    except ShapeError as exc:
        return _usage(str(exc))
    try:
        if args.output:
            with open(args.output, "w", newline="") as fh:
                write_records(records, fh, args.format, args.extended)
        else:
            write_records(records, sys.stdout, args.format, args.extended)
    except OSError as exc:
        print(f"lscan: cannot write {args.output!r}: {exc}", file=sys.stderr)
        return 3
    failed = [r for r in records if r.validated == "false"]
    for rec in failed:
        print(f"lscan: {rec.algorithm} n={rec.n}: {rec.failure}", file=sys.stderr)
    return 1 if failed else 0


def main_entry():
    sys.exit(main())
