"""Summarise ncu --set full captures of the scan kernel into profiles/:
    python scripts/ncu_summary.py <tag> gpurun_out/prof_<tag>_{i32,i64,f32,f64}.ncu-rep
writes profiles/<tag>_ncu_full_scan.json and profiles/ncu_traffic.json (per-launch
dram bytes read by bench.py's roofline.traffic)."""
import csv
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "launch__shared_mem_per_block_dynamic",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "lts__t_sectors_op_read.sum", "lts__t_sectors_op_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9}


def main():
    tag, reps = sys.argv[1], sys.argv[2:]
    summ, traffic = {}, {}
    tp = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp))
    for rep in reps:
        d = os.path.basename(rep).rsplit("_", 1)[-1].split(".")[0]
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(raw.splitlines()))
        h, u, v = rows[0], rows[1], rows[2]

        def val(k):
            return float(v[h.index(k)].replace(",", "")) * SCALE.get(u[h.index(k)], 1)

        t = val("gpu__time_duration.sum")
        tr = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
        es = 4 if d in ("i32", "f32") else 8
        n = 1 << 28
        summ[d] = {"kernel": v[h.index("Kernel Name")],
                   "metrics": {k: f"{v[h.index(k)]} {u[h.index(k)]}".strip() for k in KEYS if k in h},
                   "n": n, "algorithmic_bytes": 2 * n * es, "dram_bytes_per_launch": round(tr),
                   "traffic_over_algorithmic": round(tr / (2 * n * es), 4),
                   "achieved_gbs_under_ncu": round(tr / t / 1e9, 1)}
        traffic[f"{d}_{n}"] = round(tr)
    json.dump(summ, open(os.path.join(REPO, "profiles", f"{tag}_ncu_full_scan.json"), "w"), indent=1)
    json.dump(traffic, open(tp, "w"), indent=1)
    for d, s in summ.items():
        print(d, s["metrics"]["gpu__time_duration.sum"], s["traffic_over_algorithmic"], s["achieved_gbs_under_ncu"],
              s["metrics"].get("launch__registers_per_thread"))


if __name__ == "__main__":
    main()
