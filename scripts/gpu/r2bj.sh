#!/bin/bash
# mid-n geometry rule: byte crossovers (default) vs the capacity rule
# (LSCAN_GEOM_RULE=0), interleaved twice, graph-timed, CUB beside
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bj; mkdir -p $O
{
for rep in 1 2; do
  timeout 300 python scripts/xl_ab.py geom3
  LSCAN_GEOM_RULE=0 timeout 300 python scripts/xl_ab.py geom3
done
} 2>&1 | grep -v query > $O/geom.jsonl
python - <<'PY'
import json, collections
rows=[json.loads(l) for l in open("gpurun_out/r2bj/geom.jsonl") if l.startswith("{")]
t=collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows:
    k="bytes" if r["rule"]=="1" else "capacity"
    t[(r["dtype"],r["n"])][k].append(r["us"]); t[(r["dtype"],r["n"])]["cub"].append(r["cub_us"])
    if r.get("exact") is False: print("INEXACT", r)
for k,v in t.items(): print(k, dict(v))
PY
