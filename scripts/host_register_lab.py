"""Cost of pinning a pageable numpy buffer in place (cudaHostRegister /
cudaHostUnregister of x and y, 1 GiB each) — the alternative to staging
pageable arrays through pinned buffers in ls_scan_host.  Measured: 160 ms to
register 2 GiB and 35 ms to unregister, against 79 ms for the whole staged
pageable scan, so the staging stays."""
import time

import numpy as np
import torch


def main():
    rt = torch.cuda.cudart()
    n = 1 << 28
    x = np.random.default_rng(0).integers(-100, 100, n, dtype=np.int32)
    y = np.empty_like(x)
    torch.cuda.init()
    for _ in range(3):
        t0 = time.perf_counter()
        r1 = rt.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
        r2 = rt.cudaHostRegister(y.ctypes.data, y.nbytes, 0)
        t1 = time.perf_counter()
        rt.cudaHostUnregister(x.ctypes.data)
        rt.cudaHostUnregister(y.ctypes.data)
        t2 = time.perf_counter()
        print("register 2 GiB", round((t1 - t0) * 1e3, 1), "ms; unregister", round((t2 - t1) * 1e3, 1), "ms", r1, r2)


if __name__ == "__main__":
    main()
