"""Geometry laboratory: time the hot kernel (add) under alternative
compile-time geometries (bench_support/lscan_lab.cu, ls_lab_run) next to
torch copy_ and torch.cumsum, on one GPU.  The sweeps that chose the
production geometry are in profiles/r1_lab_ws2*.json.

    python scripts/lab.py [--n 268435456] [--cfgs 34,40] [--wide] [--labso liblscanlab.so]
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

# scanner warps / tile bytes / stages (bench_support/lscan_lab.cu)
CFG_NAMES = {30: "reg16/32K/4", 31: "reg16/32K/5", 32: "reg16/32K/6", 33: "reg16/32K/7", 34: "reg8/32K/6",
             35: "reg16/64K/3", 36: "reg16/16K/12", 37: "reg8/16K/12", 38: "reg24/48K/4", 40: "reg12/48K/4",
             41: "reg8/32K/5", 42: "reg8/32K/4", 43: "reg12/48K/3", 44: "reg16/64K/3", 45: "reg4/32K/6",
             46: "reg8/16K/4", 47: "reg4/16K/4", 48: "reg8/16K/3", 49: "reg4/8K/4", 50: "reg8/32K/2",
             51: "reg4/16K/2", 60: "reg8/32K/6/vw2", 61: "reg12/48K/4/vw2", 62: "reg16/64K/3/vw2",
             63: "reg16/32K/6/vw2", 64: "reg16/48K/4/vw2", 65: "reg12/48K/4"}


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


def effective_sm_mhz():
    """SM clock actually running (clock64 cycles over globaltimer ns, median
    over 296 blocks; bench_support/clock_probe.cu) — NVML does not report
    the sustained-load slowdown."""
    P = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", "libclockprobe.so"))
    P.clock_probe.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_longlong, ctypes.c_void_p]
    buf = torch.zeros(3 * 296, dtype=torch.int64, device="cuda")
    P.clock_probe(buf.data_ptr(), 296, 200_000, torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    v = buf.view(-1, 3).cpu()
    return round((v[:, 1].double() / v[:, 2].double() * 1e3).median().item(), 1)


def graph_ms(fn, reps):
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
    return timeit(g.replay, 3, warm=1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1 << 28)
    ap.add_argument("--cfgs", default="34,40")
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--wide", action="store_true", help="64-bit elements (same as --dtype i64)")
    ap.add_argument("--dtype", choices=["i32", "i64", "f32", "f64"], default=None)
    ap.add_argument("--op", choices=["add", "max"], default="add")
    ap.add_argument("--labso", default="liblscanlab.so", help="lab library in bench_support/_build")
    ap.add_argument("--graph", action="store_true", help="time CUDA-graph replays (device time, no host)")
    ap.add_argument("--product", action="store_true", help="also time the product call (scan.inclusive_scan)")
    ap.add_argument("--timing", action="store_true",
                    help="lab build with -DLS_LAB_TIMING=1: per-phase cycles per tile from the header pad")
    ap.add_argument("--shift", action="store_true",
                    help="shifted-window kernel: x one element past a 16-byte boundary, y aligned")
    ap.add_argument("--sustain", type=int, default=0,
                    help="report this many consecutive blocks of --reps calls per config (drift under load)")
    ap.add_argument("--data", choices=["random", "ascending"], default="random",
                    help="ascending: sorted increasing input (a running max never keeps its carry)")
    args = ap.parse_args()
    L = N.lib()
    LAB = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", args.labso))
    LAB.ls_lab_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    LAB.ls_lab_run.restype = ctypes.c_int
    n = args.n
    tok = args.dtype or ("i64" if args.wide else "i32")
    code = {"i32": 0, "i64": 1, "f32": 2, "f64": 3}[tok]
    dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}[tok]
    es = 4 if tok in ("i32", "f32") else 8
    m = n + (1 if args.shift else 0)
    if dt.is_floating_point:
        x = torch.rand(m, dtype=dt, device="cuda") * 2 - 1
    else:
        x = torch.randint(-2**31, 2**31 - 1, (m,), dtype=dt, device="cuda")
    if args.data == "ascending":
        x = torch.sort(x).values
    if args.shift:
        x = x[1:]  # 4 or 8 bytes past the allocation's (256-byte) alignment
    y = torch.empty_like(x)
    ws = torch.zeros(L.ls_workspace_bytes(N.LS_I64, n) * 8, dtype=torch.uint8, device="cuda")
    g = ctypes.c_int64(0)
    ref = torch.cumsum(x, 0, dtype=dt) if not dt.is_floating_point else torch.cumsum(x.double(), 0)
    if args.op == "max":
        ref = torch.cummax(x, 0).values
    flags = (code << 8) | ((1 << 10) if args.op == "max" else 0) | ((1 << 11) if args.shift else 0)
    res = {"n": n, "dtype": str(dt), "lib": args.labso}
    res["torch_copy_gbs"] = round(2 * n * es / (timeit(lambda: y.copy_(x), args.reps) * 1e-3) / 1e9, 1)
    res["torch_cumsum_gelems"] = round(n / (timeit(lambda: torch.cumsum(x, 0, dtype=dt, out=y),
                                                   args.reps) * 1e-3) * 1e-9, 1)
    for cfg in [int(c) for c in args.cfgs.split(",")]:
        def step():
            rc = LAB.ls_lab_run(cfg, flags, x.data_ptr(), y.data_ptr(), n, ws.data_ptr(),
                                torch.cuda.current_stream().cuda_stream, ctypes.byref(g))
            assert rc == 0, rc
        if args.sustain:
            import time
            time.sleep(3)
            blocks = [timeit(step, args.reps, warm=0) for _ in range(args.sustain)]
            res[f"cfg{cfg}_{CFG_NAMES[cfg]}_sustained_gelems"] = [round(n / (b * 1e-3) * 1e-9, 1) for b in blocks]
            res[f"cfg{cfg}_sm_mhz_after"] = effective_sm_mhz()
            continue
        if args.timing:
            step()
            torch.cuda.synchronize()
            ws[128 - 112:128].zero_()  # header pad words (bytes 16..127)
            for _ in range(args.reps):
                step()
            torch.cuda.synchronize()
            acc = ws[16:80].view(torch.int64).cpu().tolist()
            tiles = -(-n // (8192 if es == 4 else 6144)) * args.reps
            names = ["scan_wait_data", "scan_load_rowscan_barA", "scan_totals_prefix_barB", "scan_fold_store",
                     "producer_wait_free_stage", "lookback_per_tile", "lookback_repolls_per_tile"]
            res[f"cfg{cfg}_cycles_per_tile"] = {k: round(v / tiles, 2) for k, v in zip(names, acc)}
            rounds = tiles / 148
            res[f"cfg{cfg}_cycles_per_tile"]["chain_cta_lookback_per_round"] = round(acc[7] / rounds, 1)
        ms = graph_ms(step, args.reps) if args.graph else timeit(step, args.reps)
        res[f"cfg{cfg}_{CFG_NAMES[cfg]}"] = {
            "gelems": round(n / (ms * 1e-3) * 1e-9, 1), "gbs": round(2 * n * es / (ms * 1e-3) / 1e9, 1),
            "grid": g.value,
            "ok": bool(torch.equal(y, ref)) if (not dt.is_floating_point or args.op == "max")
            else bool(((y.double() - ref).abs() <= 1e-4 * torch.cumsum(x.double().abs(), 0)).all())}
    if args.product:
        from paper_1604_04815_b200 import scan as S

        def prod():
            S.inclusive_scan(x, out=y, op=args.op)
        ms = graph_ms(prod, args.reps) if args.graph else timeit(prod, args.reps)
        res["product"] = {"gelems": round(n / (ms * 1e-3) * 1e-9, 1), "us": round(ms * 1e3, 2)}
    print(json.dumps(res, indent=None if args.graph else 1))


if __name__ == "__main__":
    main()
