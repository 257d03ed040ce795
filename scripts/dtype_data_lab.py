"""Is the f32 gap to i32 at 2^28 the kernel or the data?  Times the i32 and
f32 scans on both data patterns (full-range random ints, and U[-1,1] floats),
the other pattern reinterpreted bit for bit, CUDA events over 100 calls."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402


def gelems(x, reps=100):
    y = torch.empty_like(x)
    for _ in range(5):
        S.inclusive_scan(x, out=y)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        S.inclusive_scan(x, out=y)
    b.record()
    torch.cuda.synchronize()
    return round(x.numel() / (a.elapsed_time(b) / reps * 1e-3) * 1e-9, 1)


n = 1 << 28
ints = torch.randint(-2**31, 2**31 - 1, (n,), dtype=torch.int32, device="cuda")
floats = torch.rand(n, dtype=torch.float32, device="cuda") * 2 - 1
zeros = torch.zeros(n, dtype=torch.int32, device="cuda")
res = {"i32_kernel_int_data": gelems(ints), "i32_kernel_float_bits": gelems(floats.view(torch.int32)),
       "i32_kernel_zeros": gelems(zeros),
       "f32_kernel_float_data": gelems(floats), "f32_kernel_int_bits": gelems(ints.view(torch.float32)),
       "f32_kernel_zeros": gelems(zeros.view(torch.float32))}
print(json.dumps(res))
