"""Throughput of the fused block-cyclic multi-GPU kernel with W virtual GPUs
on one B200 (W kernels on W streams, SMs split evenly) vs the single-GPU
kernel on the same total data.  Intra-device "peer" stores stand in for
NVLink, so this measures the protocol's overhead, not NVLink latency."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_1604_04815_b200 import _native as N  # noqa: E402
from paper_1604_04815_b200 import scan as S  # noqa: E402
from paper_1604_04815_b200.errors import raise_for_status  # noqa: E402
from test_cyclic_gpu import VirtualGPUs  # noqa: E402

env = (N, S, raise_for_status)
res = {}
for dt in (torch.int32, torch.int64):
    total = 1 << 28
    x = torch.randint(-1000, 1000, (total,), dtype=dt, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        S.inclusive_scan(x, y)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(20):
        S.inclusive_scan(x, y)
    b.record()
    torch.cuda.synchronize()
    res[f"{dt}_single"] = total / (a.elapsed_time(b) / 20 * 1e-3) * 1e-9
    for W in (1, 2, 4, 8):
        n = total // W
        parts = list(x.view(W, n).unbind(0))
        v = VirtualGPUs(env, W, dt, n)
        for _ in range(2):
            v(parts, spin_budget=0)
        import time
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reps = 10
        for _ in range(reps):
            v(parts, spin_budget=0)
        torch.cuda.synchronize()
        dt_s = (time.perf_counter() - t0) / reps
        res[f"{dt}_virtual{W}"] = total / dt_s * 1e-9
        v.close()
print(json.dumps(res, indent=1))
