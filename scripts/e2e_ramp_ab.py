"""(Historical: the LSCAN_HOST_RAMP switch and the ramped schedule were removed
after this measurement — both settings now run equal chunks.)
Ramped vs equal host-pipeline chunks alternated inside one process
(LSCAN_HOST_RAMP is read per call): pinned 2^28 i32 through the numpy
drop-in, 10 alternations, median per setting."""
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1604_04815_b200 as P  # noqa: E402

n = 1 << 28
x = np.random.default_rng(1).integers(-2**31, 2**31 - 1, n, dtype=np.int32)
xp = torch.empty(n, dtype=torch.int32).pin_memory()
yp = torch.empty(n, dtype=torch.int32).pin_memory()
xp.numpy()[:] = x
prob = P.ScanProblem(xp.numpy(), P.make_operator("add", "i32"), out=yp.numpy())
P.chained_scan(prob)
ts = {"1": [], "0": []}
for _ in range(10):
    for r in ("1", "0"):
        os.environ["LSCAN_HOST_RAMP"] = r
        t0 = time.perf_counter()
        P.chained_scan(prob)
        ts[r].append(time.perf_counter() - t0)
print(json.dumps({("ramp" if r == "1" else "equal"): {"median_ms": round(statistics.median(v) * 1e3, 3),
                  "min_ms": round(min(v) * 1e3, 3), "gelems": round(n / statistics.median(v) * 1e-9, 3)}
                  for r, v in ts.items()}))
