# persistent kernel at mid sizes: the occupancy grid (148 CTAs) vs the balanced
# grid (fewest CTAs with the same round count), graph-timed sweep 2^21..2^26
for b in 0 1 0 1; do
  LSCAN_BALANCED_GRID=$b LSCAN_CLUSTER_MAX_BYTES=0 timeout 600 python scripts/sweep.py --min-log 21 --max-log 26 > gpurun_out/balanced_$b.jsonl 2>&1
  python - "$b" <<'PY'
import json, sys
b = sys.argv[1]
rows = [json.loads(l) for l in open(f"gpurun_out/balanced_{b}.jsonl") if l.startswith('{"dtype"')]
print("balanced" if b == "1" else "occupancy", [(r["dtype"], r["log2n"], r["graph_gelems"]) for r in rows])
PY
done
