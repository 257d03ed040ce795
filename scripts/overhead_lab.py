"""Per-call cost of a small scan, split into host and device parts.

For i32 at a few small N: wall-clock per call of back-to-back launches
(host-bound when the kernel is short) through

* ``scan.inclusive_scan``          the public torch API (argument checks, workspace lookup)
* the bare ctypes call             ``ls_inclusive_scan`` with prebound arguments
* CUB DeviceScan::InclusiveSum     bench_support/cub_side.cu through ctypes
* ``torch.cumsum``

and the device time per call of the same launches replayed from a CUDA graph
(ours and CUB), which removes the host from the measurement.
"""
import ctypes
import json
import os
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_1604_04815_b200 import _native as N  # noqa: E402
from paper_1604_04815_b200 import scan as S  # noqa: E402


def wall_per_call(fn, reps=3000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


def graph_per_call(fn, reps=200):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    L = N.lib()
    cub = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", "libcubside.so"))
    cub.cub_inclusive_sum.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                                      ctypes.c_void_p, ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p]
    out = {}
    for lg in [int(a) for a in (sys.argv[1:] or ["10", "14", "16", "18", "20"])]:
        n = 1 << lg
        x = torch.randint(-1000, 1000, (n,), dtype=torch.int32, device="cuda")
        y = torch.empty_like(x)
        S.inclusive_scan(x, out=y)
        torch.cuda.synchronize()
        stream = torch.cuda.current_stream()
        ws = S._workspaces[(x.device.index, stream.cuda_stream)]
        args = (0, 0, x.data_ptr(), y.data_ptr(), n, None, None, ws.data_ptr(), ws.numel(), stream.cuda_stream)
        fn = L.ls_inclusive_scan
        tb = ctypes.c_size_t(0)
        cub.cub_inclusive_sum(0, x.data_ptr(), y.data_ptr(), n, None, ctypes.byref(tb), stream.cuda_stream)
        temp = torch.empty(max(tb.value, 1), dtype=torch.uint8, device="cuda")
        cargs = (0, x.data_ptr(), y.data_ptr(), n, temp.data_ptr(), ctypes.byref(tb))
        row = {
            "api_wall_us": wall_per_call(lambda: S.inclusive_scan(x, out=y)),
            "ctypes_wall_us": wall_per_call(lambda: fn(*args)),
            "cub_wall_us": wall_per_call(lambda: cub.cub_inclusive_sum(*cargs, stream.cuda_stream)),
            "cumsum_wall_us": wall_per_call(lambda: torch.cumsum(x, 0, dtype=torch.int32, out=y)),
            "graph_us": graph_per_call(lambda: S.inclusive_scan(x, out=y)),
            "cub_graph_us": graph_per_call(
                lambda: cub.cub_inclusive_sum(*cargs, torch.cuda.current_stream().cuda_stream)),
        }
        assert torch.equal(y, torch.cumsum(x, 0, dtype=torch.int32))
        out[f"2^{lg}"] = {k: round(v, 2) for k, v in row.items()}
        print(f"2^{lg}", json.dumps(out[f"2^{lg}"]), flush=True)
    print(json.dumps({"us_per_call_i32": out}))


if __name__ == "__main__":
    main()
