"""Mid-n points around the extra-large cluster geometry's range, graph-timed
(median of 5 replays), CUB beside: run once with and once without
LSCAN_NO_XL=1 to compare the XL cluster kernel with the persistent one."""
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_1604_04815_b200 import scan as S  # noqa: E402

rows = []
SETS = {"xl": (("i32", [1 << 21, 3 << 20, 7 << 19, 1 << 22]), ("f32", [3 << 20, 1 << 22]),
              ("i64", [1 << 20, 3 << 19, 7 << 18, 1 << 21]), ("f64", [3 << 19, 1 << 21])),
        "geom": (("i32", [1 << 19, 1 << 20, 1 << 21]), ("i64", [1 << 18, 1 << 19, 1 << 20]),
                 ("f64", [1 << 17, 1 << 18, 1 << 19, 1 << 20])),
        "geom2": (("i32", [1 << 18, 1 << 19, 1 << 20, 1 << 21]), ("f32", [1 << 20, 1 << 21]),
                  ("i64", [1 << 17, 1 << 18, 1 << 19, 1 << 20]), ("f64", [1 << 16, 1 << 17, 1 << 18, 1 << 19])),
        "geom3": (("i32", [1 << 20, 5 << 18, 3 << 19, 7 << 18, 1 << 21, 5 << 19, 3 << 20]),
                  ("f32", [1 << 20, 3 << 19, 1 << 21, 3 << 20]),
                  ("i64", [1 << 18, 5 << 16, 3 << 17, 7 << 16, 1 << 19, 5 << 17, 3 << 18, 1 << 20, 3 << 19]),
                  ("f64", [1 << 18, 3 << 17, 1 << 19, 3 << 18, 1 << 20, 3 << 19]))}
for tok, sizes in SETS[sys.argv[1] if len(sys.argv) > 1 else "xl"]:
    for n in sizes:
        x = bench.device_input(n, tok, n, torch)
        y = torch.empty_like(x)
        reps = max(3, min(1000, int(2e8 // (n * 8)) + 3))
        ms = bench.graph_ms(lambda: S.inclusive_scan(x, out=y), reps, 5)
        S.inclusive_scan(x, out=y)
        torch.cuda.synchronize()
        ok = bench.int_scan_exact(x, y) if tok[0] == "i" else None
        cs = bench.cub_step(tok, x, y)
        cms = bench.graph_ms(cs, reps, 5) if cs else None
        r = {"xl": os.environ.get("LSCAN_NO_XL") != "1", "geom": os.environ.get("LSCAN_CLUSTER_GEOM"),
             "max_bytes": os.environ.get("LSCAN_CLUSTER_MAX_BYTES"),
             "rule": os.environ.get("LSCAN_GEOM_RULE", "1"), "dtype": tok, "n": n, "us": round(ms * 1e3, 3),
             "cub_us": round(cms * 1e3, 3) if cms else None, "vs_cub": round(cms / ms, 3) if cms else None, "exact": ok}
        print(json.dumps(r), flush=True)
print(json.dumps({"query": {str(dt): S.query_cluster(dt) for dt in (torch.int32, torch.int64)}}))
