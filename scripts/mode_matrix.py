"""Throughput of every (dtype, operator, mode) at N = 2^28 on the persistent
kernel: inclusive / exclusive / in place x add / max / min x i32 / i64 / f32 /
f64, with the fraction of the measured HBM copy bandwidth."""
import json
import os
import sys
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import bench  # noqa: E402
sys.path.insert(0, os.path.join(REPO, "scripts"))
from lab import effective_sm_mhz  # noqa: E402  (clock64 / globaltimer probe: the SM clock actually running)
from paper_1604_04815_b200 import scan as S  # noqa: E402


def main():
    n = 1 << 28
    peak, src = bench.choose_peak(bench.copy_probes(1 << 31))
    out = {"n": n, "peak_gbs": peak, "peak_source": src}
    # MM_DTYPES=f64,i64 restricts the dtypes; MM_COOL=S idles S seconds before
    # each row (the clocks recover from the power cap between rows)
    pick = os.environ.get("MM_DTYPES")
    cool = float(os.environ.get("MM_COOL", "0"))
    names = {"i32": torch.int32, "i64": torch.int64, "f32": torch.float32, "f64": torch.float64}
    dts = [names[t] for t in pick.split(",")] if pick else list(names.values())
    out["cool_s"] = cool
    for dt in dts:
        x = (torch.randint(-2**31, 2**31 - 1, (n,), dtype=dt, device="cuda") if not dt.is_floating_point
             else torch.rand(n, dtype=dt, device="cuda") * 2 - 1)
        y = torch.empty_like(x)
        es = x.element_size()
        for op in ("add", "max", "min"):
            for mode in ("inclusive", "exclusive", "in_place"):
                if mode == "in_place":
                    z = x.clone()
                    fn = lambda: S.inclusive_scan(z, out=z, op=op)  # noqa: E731
                elif mode == "exclusive":
                    fn = lambda: S.exclusive_scan(x, out=y, op=op)  # noqa: E731
                else:
                    fn = lambda: S.inclusive_scan(x, out=y, op=op)  # noqa: E731
                if cool:
                    time.sleep(cool)
                ms = bench.time_device(fn, 30, 3, torch.cuda.current_stream())
                g = n / (ms * 1e-3) * 1e-9
                out[f"{str(dt)[6:]}_{op}_{mode}"] = {"gelems": round(g, 1),
                                                     "frac_of_measured_hbm": round(2 * es * g / peak, 4),
                                                     "sm_mhz_after": effective_sm_mhz()}
                if mode == "in_place":
                    del z
        del x, y
        torch.cuda.empty_cache()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
