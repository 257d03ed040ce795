"""Per-block event timeline of the latency (cluster) kernel at mid n (lab
build bench_support/_build/libclusterlab_tl.so, -DLS_LAB_CTIMELINE=1): when
each block's loads + row scans were done, its cluster exchange passed, its
prefix (clusters before it) was known and its stores were issued, relative
to the first block's start; graph-timed µs per call without the marks.

    python scripts/cluster_timeline.py --variant 20 --n 1048576 [--csize 16]
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

WORDS = 6
EVENTS = ["start", "rowscans", "cluster_xchg", "prefix", "stored", "dsmem_stores"]


def pct(v, q):
    v = sorted(v)
    return v[min(len(v) - 1, int(q * (len(v) - 1) + 0.5))]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variant", type=int, default=20)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--csize", type=int, default=16)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--lib", default="libclusterlab_tl.so")
    ap.add_argument("--data", default="int", choices=["int", "unit", "fullint"],
                    help="int: small integers; unit: U[-1,1] (floats); fullint: full-range ints")
    a = ap.parse_args()
    L = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", a.lib))
    L.lab_cluster.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                              ctypes.c_int, ctypes.c_void_p]
    L.lab_block_elems.restype = ctypes.c_longlong
    L.lab_set_timeline.argtypes = [ctypes.c_void_p]
    L.lab_set_cluster_size.argtypes = [ctypes.c_int]
    L.lab_set_cluster_size(a.csize)
    be = L.lab_block_elems(a.variant)  # elements of the variant's own type
    es = 8 if a.variant in (8, 9, 10, 11, 13, 14, 18, 19, 20, 22, 23, 24, 25, 26) else 4
    dt = torch.float64 if a.variant in (25, 26) else (torch.int64 if es == 8 else torch.int32)
    n = a.n
    if a.data == "unit":
        x = torch.rand(n, dtype=dt, device="cuda") * 2 - 1
    elif a.data == "fullint":
        x = torch.randint(torch.iinfo(dt).min, torch.iinfo(dt).max, (n,), dtype=dt, device="cuda")
    else:
        x = torch.randint(-1000, 1000, (n,), device="cuda").to(dt)  # integer-valued: f64 sums exact
    y = torch.empty_like(x)
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    blocks = -(-n // be)
    tl = torch.zeros(max(blocks, 1) * WORDS + 64, dtype=torch.int64, device="cuda")

    def step():
        rc = L.lab_cluster(a.variant, x.data_ptr(), y.data_ptr(), n, ws.data_ptr(), 1,
                           torch.cuda.current_stream().cuda_stream)
        assert rc == 0, rc

    L.lab_set_timeline(None)
    us = graph_ms(step, 50) * 1e3
    if a.data == "unit":
        ok = bool(((y - torch.cumsum(x, 0)).abs() <= 1e-9 * torch.cumsum(x.abs(), 0) + 1e-12).all())
    else:
        ok = bool(torch.equal(y, torch.cumsum(x, 0, dtype=dt)))  # exact for integer-valued f64 too
    if a.lib != "libclusterlab_tl.so":  # a build without the marks: graph time only
        print(json.dumps({"variant": a.variant, "n": n, "csize": a.csize, "lib": a.lib, "data": a.data,
                          "graph_us_no_marks": round(us, 3), "exact": ok}))
        return
    L.lab_set_timeline(tl.data_ptr())
    for _ in range(a.reps):
        step()
    torch.cuda.synchronize()
    v = tl[:blocks * WORDS].view(blocks, WORDS).cpu().tolist()
    t0 = min(r[0] for r in v)
    out = {"variant": a.variant, "n": n, "csize": a.csize, "data": a.data, "blocks": blocks, "graph_us_no_marks": round(us, 3),
           "exact": ok}
    for e, name in enumerate(EVENTS):
        vals = [(r[e] - t0) / 1e3 for r in v]
        out[name] = {"min": round(min(vals), 3), "p50": round(pct(vals, 0.5), 3), "p90": round(pct(vals, 0.9), 3),
                     "max": round(max(vals), 3)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
