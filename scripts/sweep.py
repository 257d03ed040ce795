"""BASELINE configs[3]: the N sweep (2^10 .. 2^30 x i32/i64/f32/f64) on one
B200, ours next to CUB DeviceScan on the same buffers, device time per call
from CUDA-graph replay (bench.graph_ms), every point validated (integers
exactly, floats by the envelope against the strict fold).  One JSON row per
point, then a summary line.

    python scripts/sweep.py [--min-log 10] [--max-log 30] [--dtypes i32,i64,f32,f64] [--logs 20,21,22]
                            [--path auto|persistent|cluster]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-log", type=int, default=10)
    ap.add_argument("--max-log", type=int, default=30)
    ap.add_argument("--logs", default=None, help="explicit comma-separated log2 sizes (overrides min/max)")
    ap.add_argument("--dtypes", default="i32,i64,f32,f64")
    ap.add_argument("--no-cub", action="store_true")
    ap.add_argument("--path", default="auto", choices=["auto", "persistent", "cluster"],
                    help="pin the kernel choice (scan.force_path)")
    a = ap.parse_args()
    S.force_path(a.path).__enter__()
    logs = [int(v) for v in a.logs.split(",")] if a.logs else list(range(a.min_log, a.max_log + 1))
    rows = []
    for tok in a.dtypes.split(","):
        for lg in logs:
            n = 1 << lg
            x = bench.device_input(n, tok, n, torch)
            y = torch.empty_like(x)
            reps = max(3, min(1000, int(2e8 // (n * 8)) + 3))
            trials = 5 if n <= (1 << 24) else 1  # median of replays where a call is short
            ms = bench.graph_ms(lambda: S.inclusive_scan(x, out=y), reps, trials)
            S.inclusive_scan(x, out=y)
            torch.cuda.synchronize()
            if tok[0] == "i":
                ok = bench.int_scan_exact(x, y)
            elif n <= (1 << 28):
                yref = torch.empty_like(x)
                S.ordered_scan(x, yref)
                ok = bench.float_envelope(x, y, yref, tok)["ok"]
                del yref
            else:
                ok = None
            row = {"dtype": tok, "path": a.path, "log2n": lg, "n": n, "us_per_call": round(ms * 1e3, 3),
                   "gelems": round(n / (ms * 1e-3) * 1e-9, 2), "validated": ok}
            cs = None if a.no_cub else bench.cub_step(tok, x, y)
            if cs is not None:
                cms = bench.graph_ms(cs, reps, trials)
                row["cub_us"] = round(cms * 1e3, 3)
                row["vs_cub"] = round(cms / ms, 3)
            rows.append(row)
            print(json.dumps(row), flush=True)
            del x, y
            torch.cuda.empty_cache()
    behind = [(r["dtype"], r["log2n"], r.get("vs_cub")) for r in rows if r.get("vs_cub") is not None and r["vs_cub"] < 1.1]
    print(json.dumps({"points": len(rows), "all_validated": all(r["validated"] in (True, None) for r in rows),
                      "below_1.10x_cub": behind}))


if __name__ == "__main__":
    main()
