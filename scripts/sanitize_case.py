"""Small scans for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402

for dt in (torch.int32, torch.float64):
    for n in (5, 8192 * 3 + 7, 300_001):
        x = (torch.arange(n, dtype=dt, device="cuda") % 7) - 3
        y = S.inclusive_scan(x)
        ref = torch.cumsum(x.double(), 0).to(dt)
        assert torch.equal(y, ref), (dt, n)
        S.exclusive_scan(x)
        x2 = x[1:]  # misaligned -> generic kernel
        S.inclusive_scan(x2)
        S.reduce_sum(x)
torch.cuda.synchronize()
print("sanitize cases ok")
