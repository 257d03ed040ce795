"""Small scans for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

    python scripts/sanitize_case.py [all|full|partial|generic|reduce|cluster|shifted]

full / partial / generic run with the persistent kernel forced (small sizes
would otherwise take the latency kernel); cluster runs the latency kernel on
one cluster, several clusters (small, mid and large tiles), misaligned
inputs and a carry.
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1604_04815_b200 import scan as S  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "all"
for dt in (torch.int32, torch.float32, torch.float64):
    if mode in ("all", "cluster"):
        c = S.query_cluster(dt)
        with S.force_path("cluster"):
            # one cluster, several (mid / large tiles), the extra-large geometry's top
            for n in (5, c["block_elems"] * 3 + 7, c["one_cluster_elems"] + 11, c["mid_max_elems"] + 5,
                      c["max_elems"] - 3):
                for off in (0, 1):
                    x = ((torch.arange(n + 1, dtype=dt, device="cuda") % 7) - 3)[off:off + n]
                    for op in ("add", "max"):
                        y = S.inclusive_scan(x, op=op)
                        ref = torch.cumsum(x.double(), 0).to(dt) if op == "add" else torch.cummax(x, 0).values
                        assert torch.equal(y, ref), (dt, n, "cluster", op)
                        S.exclusive_scan(x, op=op, carry_in=x[:1].clone())
    if mode in ("all", "shifted"):
        # misaligned x, aligned y, n >= 2^20: the shifted-window TMA kernel + latency-kernel tail
        tile = S.query_config(dt, 1 << 20)["tile_elems"]
        for n in ((1 << 20) // tile * tile + 2 * tile, (1 << 20) + 7, (1 << 20) // tile * tile + tile + 1):
            # x ends exactly at its allocation's end (no slack to over-read)
            x = ((torch.arange(n + 1, dtype=dt, device="cuda") % 7) - 3)[1:]
            y = S.inclusive_scan(x)
            if not dt.is_floating_point or dt == torch.float64:
                assert torch.equal(y, torch.cumsum(x.double(), 0).to(dt)), (dt, n, "shifted")
            S.exclusive_scan(x)
            # max with x misaligned, y aligned: the shifted kernel's second reducer (32-bit too)
            assert torch.equal(S.inclusive_scan(x, op="max"), torch.cummax(x, 0).values), (dt, n, "shifted max")
            # y misaligned the other way: head folded in the kernel
            yb = torch.empty(n + 1, dtype=dt, device="cuda")
            S.inclusive_scan(x, out=yb[1:], op="max")
            assert torch.equal(yb[1:], torch.cummax(x, 0).values), (dt, n, "shifted max")
            # congruent slices in place (x == y, head stored by the last CTA)
            # and y 16 bytes past a 32-byte boundary
            for off in (1, 16 // x.element_size()):
                z = ((torch.arange(n + off, dtype=dt, device="cuda") % 7) - 3)
                ref = torch.cumsum(z[off:].double(), 0).to(dt)
                S.inclusive_scan(z[off:], out=z[off:])
                assert torch.equal(z[off:], ref), (dt, n, "in place", off)
    if mode in ("cluster", "shifted"):
        continue
    tile = S.query_config(dt, 1 << 20)["tile_elems"]
    sizes = {"full": (tile * 3, tile * 200), "partial": (5, tile * 3 + 7, 300_001),
             "generic": (tile * 3 + 7,), "reduce": (300_001,)}
    for m, ns in sizes.items():
        if mode not in ("all", m):
            continue
        for n in ns:
            x = (torch.arange(n + 1, dtype=dt, device="cuda") % 7) - 3
            if m == "generic":
                x = x[1:]  # misaligned -> generic kernel
            else:
                x = x[:n]
            if m == "reduce":
                S.reduce_sum(x)
                continue
            with S.force_path("persistent"):
                for op in ("add", "max"):
                    y = S.inclusive_scan(x, op=op)
                    ref = torch.cumsum(x.double(), 0).to(dt) if op == "add" else torch.cummax(x, 0).values
                    assert torch.equal(y, ref), (dt, n, m, op)
                    S.exclusive_scan(x, op=op)
torch.cuda.synchronize()
print("sanitize cases ok", mode)
