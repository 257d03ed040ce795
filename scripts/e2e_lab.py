"""End-to-end host-array scans through the numpy drop-in (pinned and
pageable 2^28 i32), wall time per call, median of 7 — for A/B of the host
pipeline (e.g. LSCAN_HOST_RAMP=0, LSCAN_HOST_CHUNK_MB=16)."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_04815_b200 as P  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 28
x = np.random.default_rng(n).integers(-2**31, 2**31 - 1, n, dtype=np.int32)
xp = torch.empty(n, dtype=torch.int32).pin_memory()
yp = torch.empty(n, dtype=torch.int32).pin_memory()
xp.numpy()[:] = x
op = P.make_operator("add", "i32")
res = {"n": n, "ramp": os.environ.get("LSCAN_HOST_RAMP", "1"), "chunk_mb": os.environ.get("LSCAN_HOST_CHUNK_MB", "32")}
for name, xs, ys in (("pinned", xp.numpy(), yp.numpy()), ("pageable", x, np.empty_like(x))):
    prob = P.ScanProblem(xs, op, out=ys)
    P.chained_scan(prob)
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        P.chained_scan(prob)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    res[name] = {"ms": round(t * 1e3, 3), "gelems": round(n / t * 1e-9, 3),
                 "exact": bool(np.array_equal(ys[-1000:], np.cumsum(x, dtype=np.int32)[-1000:]))}
print(json.dumps(res))
