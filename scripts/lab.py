"""Kernel laboratory: time the i32 scan under alternative geometries and
experiment flags (ls_lab_run), next to torch copy_ and CUB, on one GPU.

    python scripts/lab.py [--n 268435456] [--cfgs 0,1,2] [--reps 50] [--ncu]
"""

import argparse
import ctypes
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from paper_1604_04815_b200 import _native as N  # noqa: E402

CFG_NAMES = {0: "512t/32K/6st", 1: "512t/32K/4st", 2: "512t/16K/12st", 3: "1024t/64K/3st",
             4: "256t/16K/6st(2/SM)", 5: "512t/32K/3st(2/SM)", 6: "256t/32K/6st(V8)",
             10: "ws16/32K/6", 11: "ws16/32K/4", 12: "ws8/32K/6", 13: "ws16/64K/3", 14: "ws32/64K/3",
             15: "ws8/16K/12", 16: "ws16/16K/12", 17: "ws16/32K/7", 18: "ws8/32K/7", 19: "ws16/64K/3",
             20: "ws16/32K/5", 30: "reg16/32K/4", 31: "reg16/32K/5", 32: "reg16/32K/6", 33: "reg16/32K/7",
             34: "reg8/32K/6", 35: "reg16/64K/3", 36: "reg16/16K/12", 37: "reg8/16K/12", 38: "reg24/48K/4",
             39: "ws16/32K/6", 40: "reg12/48K/4", 41: "reg8/32K/5", 42: "reg8/32K/4"}


def timeit(fn, reps, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--cfgs", default=",".join(str(k) for k in CFG_NAMES))
    ap.add_argument("--flags", default="0,1")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--ncu", action="store_true", help="few launches of cfg 0 only (for profiling)")
    ap.add_argument("--wide", action="store_true", help="64-bit elements (ws/ws2 configs)")
    ap.add_argument("--labso", default="liblscanlab.so", help="lab library in bench_support/_build")
    args = ap.parse_args()
    L = N.lib()
    LAB = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", args.labso))
    LAB.ls_lab_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                             ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    LAB.ls_lab_run.restype = ctypes.c_int
    n = args.n
    dt = torch.int64 if args.wide else torch.int32
    es = 8 if args.wide else 4
    x = torch.randint(-2**31, 2**31 - 1, (n,), dtype=dt, device="cuda")
    y = torch.empty_like(x)
    wsb = L.ls_workspace_bytes(N.LS_I64, n) * 8
    ws = torch.zeros(wsb, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    g = ctypes.c_int64(0)
    ref = torch.cumsum(x, 0, dtype=dt)
    if args.ncu:
        for _ in range(4):
            assert LAB.ls_lab_run(0, 0, x.data_ptr(), y.data_ptr(), n, ws.data_ptr(), s, ctypes.byref(g)) == 0
        torch.cuda.synchronize()
        return
    res = {"n": n}
    res["torch_copy_gbs"] = round(2 * n * es / (timeit(lambda: y.copy_(x), args.reps) * 1e-3) / 1e9, 1)
    res["torch_cumsum_gelems"] = round(n / (timeit(lambda: torch.cumsum(x, 0, dtype=dt, out=y),
                                                   args.reps) * 1e-3) * 1e-9, 1)
    for cfg in [int(c) for c in args.cfgs.split(",")]:
        for fl in [int(f) for f in args.flags.split(",")]:
            def step():
                rc = LAB.ls_lab_run(cfg, fl | (256 if args.wide else 0), x.data_ptr(), y.data_ptr(), n, ws.data_ptr(), s, ctypes.byref(g))
                assert rc == 0, rc
            ms = timeit(step, args.reps)
            ok = None
            if fl == 0 or cfg >= 10:
                ok = bool(torch.equal(y, ref))
            res[f"cfg{cfg}_{CFG_NAMES[cfg]}_flags{fl}"] = {
                "gelems": round(n / (ms * 1e-3) * 1e-9, 1), "gbs": round(2 * n * es / (ms * 1e-3) / 1e9, 1),
                "grid": g.value, "ok": ok}
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
