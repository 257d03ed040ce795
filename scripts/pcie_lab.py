"""PCIe ceiling for the e2e path: pinned H2D alone, D2H alone, both at once,
and the host-buffer scan pipeline at several chunk sizes (subprocesses, since
the chunk size is read once per process)."""
import json
import os
import subprocess
import sys
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
    if len(sys.argv) > 1 and sys.argv[1] == "pipe":
        sys.path.insert(0, REPO)
        import numpy as np
        import paper_1604_04815_b200 as P
        n = 1 << 28
        xp = torch.randint(-100, 100, (n,), dtype=torch.int32).pin_memory()
        yp = torch.empty(n, dtype=torch.int32).pin_memory()
        prob = P.ScanProblem(xp.numpy(), P.make_operator("add", "i32"), out=yp.numpy())
        t = timed(lambda: P.chained_scan(prob))
        xu = np.random.default_rng(0).integers(-100, 100, n, dtype=np.int32)
        tu = timed(lambda: P.chained_scan(P.ScanProblem(xu, P.make_operator("add", "i32"))), reps=3)
        print(json.dumps({"chunk_mb": os.environ.get("LSCAN_HOST_CHUNK_MB"), "pinned_ms": t * 1e3,
                          "pinned_gelems": n / t * 1e-9, "pageable_ms": tu * 1e3, "pageable_gelems": n / tu * 1e-9}))
        return
    nbytes = 1 << 30
    h1 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    h2 = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    d1 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {}
    res["h2d_gbs"] = nbytes / timed(lambda: d1.copy_(h1, non_blocking=True)) / 1e9
    res["d2h_gbs"] = nbytes / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9

    def both():
        with torch.cuda.stream(s1):
            d1.copy_(h1, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    res["bidir_each_gbs"] = nbytes / timed(both) / 1e9
    out = [res]
    for mb in (8, 16, 32, 64, 128):
        env = dict(os.environ, LSCAN_HOST_CHUNK_MB=str(mb))
        r = subprocess.run([sys.executable, __file__, "pipe"], env=env, capture_output=True, text=True, timeout=300)
        out.append(json.loads(r.stdout.strip().splitlines()[-1]) if r.returncode == 0 else {"mb": mb, "err": r.stderr[-300:]})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
