"""Per-CTA event timeline of the persistent kernel (lab build with
-DLS_LAB_TIMELINE=1, bench_support/_build/liblscanlab_timeline.so): when each
CTA's k-th tile landed, its aggregate was published, its prefix was known
and its stores were issued, relative to the first CTA's start (%globaltimer).
Shows where a mid-n call spends its time (the round chain, the ring fill
order, the scan itself).

    python scripts/timeline_lab.py --dtype i32 --n 4194304 [--cfg 60]
"""
import argparse
import ctypes
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "scripts"))
from lab import graph_ms  # noqa: E402

from paper_1604_04815_b200 import _native as N  # noqa: E402

WORDS = 66  # kTimelineWords (lscan_scan_ws2.cuh)
EVENTS = ["landed", "published", "prefix", "stored", "lb_start", "lb_first_pass"]


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * (len(v) - 1) + 0.5))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="i32", choices=["i32", "i64", "f32", "f64"])
    ap.add_argument("--n", type=int, default=1 << 22)
    ap.add_argument("--cfg", type=int, default=None)
    ap.add_argument("--labso", default="liblscanlab_timeline.so")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    cfg = a.cfg if a.cfg is not None else {"i32": 60, "i64": 61, "f32": 65, "f64": 61}[a.dtype]
    L = N.lib()
    LAB = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", a.labso))
    LAB.ls_lab_run.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64,
                               ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
    LAB.ls_lab_set_timeline.argtypes = [ctypes.c_void_p]
    code = {"i32": 0, "i64": 1, "f32": 2, "f64": 3}[a.dtype]
    dt = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}[a.dtype]
    x = (torch.randint(-2**31, 2**31 - 1, (a.n,), dtype=dt, device="cuda") if not dt.is_floating_point
         else torch.rand(a.n, dtype=dt, device="cuda"))
    y = torch.empty_like(x)
    ws = torch.zeros(L.ls_workspace_bytes(N.LS_I64, a.n) * 8, dtype=torch.uint8, device="cuda")
    tl = torch.zeros(1024 * WORDS, dtype=torch.int64, device="cuda")
    g = ctypes.c_int64(0)
    flags = code << 8

    def step():
        rc = LAB.ls_lab_run(cfg, flags, x.data_ptr(), y.data_ptr(), a.n, ws.data_ptr(),
                            torch.cuda.current_stream().cuda_stream, ctypes.byref(g))
        assert rc == 0, rc

    LAB.ls_lab_set_timeline(None)
    us = graph_ms(step, 50) * 1e3
    ok = bool(torch.equal(y, torch.cumsum(x, 0, dtype=dt))) if not dt.is_floating_point else None
    LAB.ls_lab_set_timeline(tl.data_ptr())
    for _ in range(a.reps):
        step()
    torch.cuda.synchronize()
    G = g.value
    v = tl[:G * WORDS].view(G, WORDS).cpu().tolist()
    t0 = min(r[0] for r in v)
    rel = [[((w - t0) / 1e3 if w else None) if not (i >= 2 and (i - 2) % 8 == 6) else w for i, w in enumerate(r)]
           for r in v]
    out = {"dtype": a.dtype, "n": a.n, "cfg": cfg, "grid": G, "graph_us_no_marks": round(us, 3),
           "exact": ok, "start_spread_us": round(max(r[0] for r in rel), 3),
           "end": {"p50": round(pct([r[1] for r in rel], 0.5), 3), "max": round(max(r[1] for r in rel), 3)}}
    ticks = sorted({w for r in v for i, w in enumerate(r) if w and not (i >= 2 and (i - 2) % 8 == 6)})
    diffs = [b - c for b, c in zip(ticks[1:], ticks[:-1]) if b != c]
    out["timer_min_step_ns"] = min(diffs) if diffs else None
    for k in range(8):
        row = {}
        for e, name in enumerate(EVENTS):
            vals = [r[2 + 8 * k + e] for r in rel if r[2 + 8 * k + e] is not None]
            if vals:
                row[name] = {"min": round(min(vals), 3), "p50": round(pct(vals, 0.5), 3),
                             "p90": round(pct(vals, 0.9), 3), "max": round(max(vals), 3), "ctas": len(vals)}
        polls = [r[2 + 8 * k + 6] for r in rel if r[2 + 8 * k + 2] is not None]
        if polls:
            row["polls"] = {"p50": pct(polls, 0.5), "max": max(polls)}
        if row:
            out[f"tile{k}"] = row
    print(json.dumps(out))


if __name__ == "__main__":
    main()
