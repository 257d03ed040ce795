"""Small-N cost of the cooperative launch vs a plain launch of the same
scan (LSCAN_NO_COOP=1 in a subprocess), graph-timed."""
import json
import os
import subprocess
import sys

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run():
    sys.path.insert(0, REPO)
    from paper_1604_04815_b200 import scan as S
    out = {}
    for lg in (10, 14, 18, 20, 22, 24):
        n = 1 << lg
        x = torch.randint(-9, 9, (n,), dtype=torch.int32, device="cuda")
        y = torch.empty_like(x)
        S.inclusive_scan(x, y)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            S.inclusive_scan(x, y)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(100):
                    S.inclusive_scan(x, y)
        g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.replay()
        b.record()
        torch.cuda.synchronize()
        out[lg] = round(a.elapsed_time(b) / 100 * 1e3, 2)
        assert torch.equal(y, torch.cumsum(x, 0, dtype=torch.int32))
    print(json.dumps(out))


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run()
    else:
        res = {}
        for coop in ("1", "0"):
            env = dict(os.environ, LSCAN_NO_COOP="0" if coop == "1" else "1")
            r = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
            res["cooperative" if coop == "1" else "plain"] = json.loads(r.stdout.strip().splitlines()[-1]) \
                if r.returncode == 0 else r.stderr[-400:]
        print(json.dumps({"us_per_call": res}, indent=1))
