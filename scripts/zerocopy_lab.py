"""Zero-copy PCIe laboratory: GB/s of SM loads/stores on pinned host memory
(bench_support/zerocopy_lab.cu) against the DMA engines (torch copies), one
direction and both at once, at a few grid sizes.  Decides whether a scan that
reads x from and writes y to host memory directly could beat the staged
pipeline of ls_scan_host (profiles/r1_pcie_e2e.json)."""
import ctypes
import json
import os
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return sorted(ts)[len(ts) // 2]


def main():
    L = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", "libzerocopylab.so"))
    L.zc_devptr.restype = ctypes.c_void_p
    L.zc_devptr.argtypes = [ctypes.c_void_p]
    L.zc_run.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t,
                         ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    nbytes = 1 << 30
    hin = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    hout = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    dev2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    din = L.zc_devptr(hin.data_ptr())
    dout = L.zc_devptr(hout.data_ptr())
    res = {"devptr_equals_hostptr": din == hin.data_ptr() and dout == hout.data_ptr()}
    s = torch.cuda.current_stream().cuda_stream
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res["dma_h2d_gbs"] = nbytes / timed(lambda: dev.copy_(hin, non_blocking=True)) / 1e9
    res["dma_d2h_gbs"] = nbytes / timed(lambda: hout.copy_(dev, non_blocking=True)) / 1e9

    def dma_both():
        with torch.cuda.stream(s1):
            dev.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(dev2, non_blocking=True)
    res["dma_both_gbs_each"] = nbytes / timed(dma_both) / 1e9
    for grid in (148, 296, 592, 1184):
        for threads in (256, 512):
            k = f"g{grid}_t{threads}"
            res[f"zc_read_{k}"] = nbytes / timed(lambda: L.zc_run(0, din, dout, dev.data_ptr(), nbytes, grid,
                                                                  threads, s)) / 1e9
            res[f"zc_write_{k}"] = nbytes / timed(lambda: L.zc_run(1, din, dout, dev.data_ptr(), nbytes, grid,
                                                                   threads, s)) / 1e9
            res[f"zc_both_{k}"] = nbytes / timed(lambda: L.zc_run(2, din, dout, dev.data_ptr(), nbytes, grid,
                                                                  threads, s)) / 1e9
    torch.cuda.synchronize()
    hin[: 1 << 20].random_(0, 255)
    L.zc_run(2, din, dout, dev.data_ptr(), 1 << 20, 148, 256, s)
    torch.cuda.synchronize()
    res["zc_both_correct"] = bool(torch.equal(hin[: 1 << 20], hout[: 1 << 20]))
    print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in res.items()}, indent=1))


if __name__ == "__main__":
    main()
