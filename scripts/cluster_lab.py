"""Graph-timed latency of the small-n kernel variants in
bench_support/cluster_lab.cu (i32, one cluster per call) next to the
product path and CUB, to choose the latency kernel's geometry."""
import ctypes
import json
import os
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "scripts"))
from overhead_lab import graph_per_call  # noqa: E402

from paper_1604_04815_b200 import scan as S  # noqa: E402

NAMES = {0: "scan_256x4", 1: "scan_512x4", 2: "scan_256x8", 3: "scan_256x2", 4: "copy_1024x4", 5: "copy_256x4",
         6: "scan_256x16_minb2", 7: "scan_256x8_minb2", 8: "i64_256x4", 9: "i64_256x8_minb2",
         10: "i64_512x4_minb2", 11: "i64_512x2", 12: "scan_256x16_minb1", 13: "i64_256x16_minb1",
         14: "i64_256x12_minb2", 15: "scan_256x12_minb2", 16: "vw2_256x4", 17: "vw2_256x8_minb2",
         18: "vw2_i64_256x4", 19: "vw2_i64_256x8_minb2", 20: "vw2_i64_256x12_minb2", 21: "vw2_256x12_minb2",
         22: "vw2_i64_512x4_minb2", 23: "vw2_i64_512x8_minb1", 24: "vw2_i64_512x6_minb1"}
WIDE = {8, 9, 10, 11, 13, 14, 18, 19, 20, 22, 23, 24}


def main():
    L = ctypes.CDLL(os.path.join(REPO, "bench_support", "_build", "libclusterlab.so"))
    L.lab_cluster.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_void_p,
                              ctypes.c_int, ctypes.c_void_p]
    L.lab_block_elems.restype = ctypes.c_longlong
    out = {}
    ws = torch.zeros(1 << 22, dtype=torch.uint8, device="cuda")
    for lg in [int(a) for a in os.environ.get("LAB_LOGS", "10,12,14,16,17,18,19,20,21,22").split(",")]:
        n = 1 << lg
        x32 = torch.randint(-1000, 1000, (n,), dtype=torch.int32, device="cuda")
        x64 = x32.long()
        y32, y64 = torch.empty_like(x32), torch.empty_like(x64)
        x, y = x32, y32
        row = {"product_us": round(graph_per_call(lambda: S.inclusive_scan(x32, out=y32)), 2),
               "product_i64_us": round(graph_per_call(lambda: S.inclusive_scan(x64, out=y64)), 2)}
        only = os.environ.get("LAB_VARIANTS")
        for v, name in NAMES.items():
            if only and str(v) not in only.split(","):
                continue
            x, y = (x64, y64) if v in WIDE else (x32, y32)
            for coop in (1,):
                tiles = -(-n // L.lab_block_elems(v))
                if (v in (4, 5) and tiles > 16) or (coop == 0 and tiles <= 16) or tiles > 16 * 24:
                    continue
                # a grid that cannot be co-resident is refused at launch: skip it
                rc = L.lab_cluster(v, x.data_ptr(), y.data_ptr(), n, ws.data_ptr(), coop,
                                   torch.cuda.current_stream().cuda_stream)
                torch.cuda.synchronize()
                if rc != 0:
                    continue

                def f(v=v, coop=coop, x=x, y=y):
                    rc = L.lab_cluster(v, x.data_ptr(), y.data_ptr(), n, ws.data_ptr(), coop,
                                       torch.cuda.current_stream().cuda_stream)
                    assert rc == 0, rc
                key = name + ("" if coop else "_nocoop") + "_us"
                row[key] = round(graph_per_call(f), 2)
                if v not in (4, 5):
                    f()
                    torch.cuda.synchronize()
                    assert torch.equal(y, torch.cumsum(x, 0, dtype=x.dtype)), name
        out[f"2^{lg}"] = row
        print(f"2^{lg}", json.dumps(row), flush=True)
    print(json.dumps({"cluster_lab_graph_us": out}))


if __name__ == "__main__":
    main()
