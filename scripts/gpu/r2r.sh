#!/bin/bash
# cluster (latency) kernel timelines at mid n, 16- and 8-block clusters
cd "$(dirname "$0")/../.."
O=gpurun_out/r2r; mkdir -p $O
for cs in 16; do
  for spec in "19 131072" "19 262144" "20 524288" "20 1048576" "7 524288" "15 1048576" "15 2097152" "0 65536"; do
    set -- $spec
    timeout 120 python scripts/cluster_timeline.py --variant $1 --n $2 --csize $cs >> $O/ctl.jsonl 2>&1
  done
done
