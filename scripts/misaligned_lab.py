"""Throughput of the non-congruent misaligned cases at 2^28 (x offset by one
element and y aligned, the reverse, and x / y at different offsets; add and
max): the generic head + shifted-window path of ls_inclusive_scan."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402


def rate(x, y, reps=20, op="add"):
    for _ in range(3):
        S.inclusive_scan(x, out=y, op=op)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        S.inclusive_scan(x, out=y, op=op)
    b.record()
    torch.cuda.synchronize()
    return round(x.numel() / (a.elapsed_time(b) / reps * 1e-3) * 1e-9, 1)


n = 1 << 28
for dt in (torch.int32, torch.int64, torch.float32, torch.float64):
    big = torch.randint(-1000, 1000, (n + 4,), device="cuda").to(dt)
    out = torch.empty(n + 4, dtype=dt, device="cuda")
    res = {"aligned": rate(big[:n], out[:n])}
    for xo, yo in ((1, 0), (0, 1), (3, 2), (1, 1)):
        res[f"x+{xo}/y+{yo}"] = rate(big[xo:xo + n], out[yo:yo + n])
    res["max x+1/y+0"] = rate(big[1:n + 1], out[:n], op="max")
    res["max x+0/y+1"] = rate(big[:n], out[1:n + 1], op="max")
    # a congruent slice scanned in place (x == y, 4 bytes past a boundary)
    res["in place x+1"] = rate(out[1:n + 1], out[1:n + 1])
    if not dt.is_floating_point:
        S.inclusive_scan(big[:n], out=out[1:n + 1])
        res["exact"] = bool(torch.equal(out[1:n + 1], torch.cumsum(big[:n], 0).to(dt)))
    print(str(dt).replace("torch.", ""), res, flush=True)
