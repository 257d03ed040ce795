"""BASELINE config 4: N sweep 2^10..2^30 x 4 dtypes on one B200, ours vs CUB.

Each point: back-to-back launches on one stream timed with CUDA events
(includes the per-call host overhead of the ctypes path), and the same
launches captured in a CUDA graph (device time only) when capture works.
Small N is L2-resident (inputs < 126 MB): those points are latency/L2-bound,
not HBM-bound; the HBM fraction is reported only where 2*N*sizeof(T) > 256 MB.
"""
import argparse
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_1604_04815_b200 import scan as S  # noqa: E402

TDT = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}


def time_events(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def time_graph(fn, reps):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()  # workspace allocation happens outside capture
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log", type=int, default=10)
    ap.add_argument("--max-log", type=int, default=30)
    ap.add_argument("--dtypes", default="i32,i64,f32,f64")
    ap.add_argument("--no-graph", action="store_true")
    a = ap.parse_args()
    peak, _ = bench.peaks()
    rows = []
    for tok in a.dtypes.split(","):
        es = 4 if tok in ("i32", "f32") else 8
        for lg in range(a.min_log, a.max_log + 1):
            n = 1 << lg
            x = torch.from_numpy(bench.synthetic(n, tok, [0, n])).cuda() if lg <= 26 else \
                (torch.randint(-2**31, 2**31 - 1, (n,), dtype=TDT[tok], device="cuda") if tok[0] == "i"
                 else torch.rand(n, dtype=TDT[tok], device="cuda") * 2 - 1)
            y = torch.empty_like(x)
            reps = 200 if lg <= 20 else (50 if lg <= 26 else 10)
            ms = time_events(lambda: S.inclusive_scan(x, out=y), reps)
            gms = None
            if not a.no_graph:
                try:
                    gms = time_graph(lambda: S.inclusive_scan(x, out=y), reps)
                except Exception as e:  # cooperative launches may not be capturable
                    gms = None
                    graph_err = str(e)[:200]
            cub = bench.cub_gelems(tok, x, reps, 3)
            cub_g = None
            if not a.no_graph:
                try:
                    cub_g = bench.cub_gelems(tok, x, reps, 3, graph=True)
                except Exception:
                    cub_g = None
            hbm = 2 * n * es > (256 << 20)
            row = {"dtype": tok, "log2n": lg, "n": n, "ms": round(ms, 5),
                   "gelems": round(n / (ms * 1e-3) * 1e-9, 2),
                   "graph_ms": None if gms is None else round(gms, 5),
                   "graph_gelems": None if gms is None else round(n / (gms * 1e-3) * 1e-9, 2),
                   "cub_gelems": None if cub is None else round(cub, 2),
                   "cub_graph_gelems": None if cub_g is None else round(cub_g, 2),
                   "frac_of_measured_hbm": round(2 * n * es / (ms * 1e-3) / 1e9 / peak, 4) if hbm else None}
            rows.append(row)
            print(json.dumps(row), flush=True)
            del x, y
            torch.cuda.empty_cache()
    print(json.dumps({"sweep": rows}))


if __name__ == "__main__":
    main()
