"""HBM ceiling lab: every copy probe of bench_support/copy_probe.cu, torch
copy_ and the i32 scan on the same 1 GiB / 2 GiB buffers (CUDA events).

    python scripts/ceiling_probe.py [--mib 1024] [--reps 20]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=1024)
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    L = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", "libcopyprobe.so"))
    for f in ("probe_tma_copy", "probe_memcpy"):
        getattr(L, f).argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
    L.probe_vec_copy.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
    L.probe_read.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
    nbytes = a.mib << 20
    x = torch.randint(0, 255, (nbytes,), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream

    def timed(fn, reps):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e-3

    res = {}
    for name, fn, mult in (
        ("tma_copy", lambda: L.probe_tma_copy(x.data_ptr(), y.data_ptr(), nbytes, s), 2),
        ("vec_copy_b2", lambda: L.probe_vec_copy(x.data_ptr(), y.data_ptr(), nbytes, 2, s), 2),
        ("vec_copy_b4", lambda: L.probe_vec_copy(x.data_ptr(), y.data_ptr(), nbytes, 4, s), 2),
        ("vec_copy_b8", lambda: L.probe_vec_copy(x.data_ptr(), y.data_ptr(), nbytes, 8, s), 2),
        ("memcpy_d2d", lambda: L.probe_memcpy(x.data_ptr(), y.data_ptr(), nbytes, s), 2),
        ("torch_copy", lambda: y.copy_(x), 2),
        ("read_b4", lambda: L.probe_read(x.data_ptr(), nbytes, sink.data_ptr(), 4, s), 1),
        ("read_b8", lambda: L.probe_read(x.data_ptr(), nbytes, sink.data_ptr(), 8, s), 1),
    ):
        t = timed(fn, a.reps)
        ts = timed(fn, max(a.reps, int(1.0 / t)))  # about a second back to back
        res[name] = {"burst_gbs": round(mult * nbytes / t / 1e9, 1), "sustained_gbs": round(mult * nbytes / ts / 1e9, 1)}
        assert name == "torch_copy" or fn() == 0
    assert torch.equal(x, y)
    from paper_1604_04815_b200 import scan as S
    xi = x.view(torch.int32)
    yi = y.view(torch.int32)
    t = timed(lambda: S.inclusive_scan(xi, out=yi), a.reps)
    ts = timed(lambda: S.inclusive_scan(xi, out=yi), int(1.0 / t))
    res["scan_i32"] = {"burst_gbs": round(2 * nbytes / t / 1e9, 1), "sustained_gbs": round(2 * nbytes / ts / 1e9, 1),
                       "gelems_burst": round(xi.numel() / t / 1e9, 1)}
    print(json.dumps({"mib": a.mib, "probes": res}))


if __name__ == "__main__":
    main()
