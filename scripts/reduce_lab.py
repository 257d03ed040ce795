"""Time the pieces of the sharded step at world size 1: reduce, carry, scan."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402


def t(fn, reps=50):
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


out = {}
for dt in (torch.int32, torch.int64):
    n = 1 << 28
    x = torch.randint(-1000, 1000, (n,), dtype=dt, device="cuda")
    y = torch.empty_like(x)
    tot = torch.empty(1, dtype=dt, device="cuda")
    totals = torch.zeros(8, dtype=dt, device="cuda")
    es = x.element_size()
    r = t(lambda: S.reduce_sum(x, tot))
    c = t(lambda: S.carry_from_totals(totals, 5))
    sc = t(lambda: S.inclusive_scan(x, y, carry_in=tot))
    ts = t(lambda: torch.sum(x))
    out[str(dt)] = {"reduce_ms": r, "reduce_read_gbs": n * es / r / 1e6, "carry_ms": c, "scan_ms": sc,
                    "torch_sum_ms": ts, "step_est_ms": r + c + sc}
print(json.dumps(out, indent=1))
