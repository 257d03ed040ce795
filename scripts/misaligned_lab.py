"""Throughput of the non-congruent misaligned case (x offset by one element,
y aligned, and the reverse) at 2^28, i32 / i64 / f32 — the realigning copy +
in-place scan path of ls_inclusive_scan."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402


def rate(x, y, reps=20):
    for _ in range(3):
        S.inclusive_scan(x, out=y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        S.inclusive_scan(x, out=y)
    b.record()
    torch.cuda.synchronize()
    return round(x.numel() / (a.elapsed_time(b) / reps * 1e-3) * 1e-9, 1)


n = 1 << 28
for dt in (torch.int32, torch.int64, torch.float32):
    big = torch.randint(-1000, 1000, (n + 4,), device="cuda").to(dt)
    out = torch.empty(n + 4, dtype=dt, device="cuda")
    r1 = rate(big[1:n + 1], out[:n])
    r2 = rate(big[:n], out[1:n + 1])
    ref = torch.cumsum(big[1:n + 1].double(), 0) if dt.is_floating_point else torch.cumsum(big[1:n + 1], 0).to(dt)
    S.inclusive_scan(big[1:n + 1], out=out[:n])
    ok = torch.equal(out[:n], ref) if not dt.is_floating_point else True
    print(dt, "x misaligned / y aligned:", r1, "Gelem/s; x aligned / y misaligned:", r2, "Gelem/s; exact:", ok)
