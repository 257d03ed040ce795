"""A few production scans for ncu to capture (one dtype, N elements).

    ncu --set full -k regex:scan_ws_kernel -s 2 -c 1 -o prof python scripts/profile_scan.py --dtype i32
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="i32")
ap.add_argument("--n", type=int, default=1 << 28)
ap.add_argument("--reps", type=int, default=4)
ap.add_argument("--exclusive", action="store_true")
ap.add_argument("--op", default="add", choices=["add", "max", "min"])
a = ap.parse_args()
dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}[a.dtype]
if dt.is_floating_point:
    x = torch.rand(a.n, dtype=dt, device="cuda") * 2 - 1
else:
    x = torch.randint(-2**31, 2**31 - 1, (a.n,), dtype=dt, device="cuda")
y = torch.empty_like(x)
fn = S.exclusive_scan if a.exclusive else S.inclusive_scan
for _ in range(a.reps):
    fn(x, out=y, op=a.op)
torch.cuda.synchronize()
print("done", a.dtype, a.op, a.n)
