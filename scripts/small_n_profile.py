"""A few scans at small/mid N for an ncu launch list (device durations)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402

for lg in (13, 16, 20, 22, 24):
    x = torch.randint(-9, 9, (1 << lg,), dtype=torch.int32, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        S.inclusive_scan(x, y)
torch.cuda.synchronize()
