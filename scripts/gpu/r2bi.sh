#!/bin/bash
# mid-n geometry choice: default vs forced cluster geometries 1/2/3 vs the
# persistent kernel (LSCAN_CLUSTER_MAX_BYTES=0), graph-timed, CUB beside
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bi; mkdir -p $O
{
timeout 300 python scripts/xl_ab.py geom2
for g in 1 2 3; do LSCAN_CLUSTER_GEOM=$g timeout 300 python scripts/xl_ab.py geom2; done
LSCAN_CLUSTER_MAX_BYTES=0 timeout 300 python scripts/xl_ab.py geom2
} 2>&1 | grep -v query > $O/geom.jsonl
python - <<'PY'
import json, collections
rows=[json.loads(l) for l in open("gpurun_out/r2bi/geom.jsonl") if l.startswith("{")]
t=collections.defaultdict(dict)
for r in rows:
    k="persist" if r.get("max_bytes")=="0" else ("g"+r["geom"] if r.get("geom") else "auto")
    t[(r["dtype"],r["n"])][k]=r["us"]; t[(r["dtype"],r["n"])]["cub"]=r["cub_us"]
for k,v in t.items(): print(k, v)
PY
