"""Throughput drift under sustained load and the SM clock behind it.

For each workload — torch copy_ of 2 GiB, CUB DeviceScan, our scan (i32 and
i64), all at N = 2^28 — 12 blocks of 50 back-to-back calls timed with CUDA
events, then the SM clock the GPU is really running (clock64 cycles over
%globaltimer ns on every SM, bench_support/clock_probe.cu; NVML keeps
reporting the maximum clock and no throttle reason).  3 s idle between
workloads so each starts from the same state."""
import ctypes
import json
import os
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
from paper_1604_04815_b200 import scan as S  # noqa: E402

P = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", "libclockprobe.so"))
P.clock_probe.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]
_buf = torch.zeros(3 * 296, dtype=torch.int64, device="cuda")


def sm_mhz():
    P.clock_probe(_buf.data_ptr(), 296, 200_000, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    v = _buf.view(-1, 3).cpu()
    return round((v[:, 1].double() / v[:, 2].double() * 1e3).median().item(), 1)


def blocks(fn, nb=12, k=50):
    evs = []
    for _ in range(nb):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            fn()
        b.record()
        evs.append((a, b))
    mhz = sm_mhz()
    return [a.elapsed_time(b) / k for a, b in evs], mhz


def main():
    n = 1 << 28
    out = {"sm_mhz_idle": sm_mhz()}
    for dt, tok in ((torch.int32, "i32"), (torch.int64, "i64")):
        x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=dt, device="cuda")
        y = torch.empty_like(x)
        es = x.element_size()
        runs = [("copy_gbs", lambda: y.copy_(x), lambda ms: 2 * n * es / (ms * 1e-3) / 1e9),
                ("ours_gelems", lambda: S.inclusive_scan(x, out=y), lambda ms: n / (ms * 1e-3) * 1e-9)]
        for name, fn, conv in runs:
            fn()
            time.sleep(3)
            ms, mhz = blocks(fn)
            out[f"{tok}_{name}"] = {"per_block": [round(conv(m), 1) for m in ms], "sm_mhz_after": mhz}
        time.sleep(3)
        per = [round(bench.cub_gelems(tok, x, 50, 0), 1) for _ in range(12)]
        out[f"{tok}_cub_gelems"] = {"per_block": per, "sm_mhz_after": sm_mhz()}
        del x, y
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
