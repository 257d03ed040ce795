#!/bin/bash
# f64 vs i64 on the latency kernel's mid geometry at 2^17 / 2^18 (f64 measured ~1 us slower
# in some sweeps): timelines and graph time, three processes each
cd "$(dirname "$0")/../.."
O=gpurun_out/r2aa; mkdir -p $O
for rep in 1 2 3; do
  for spec in "19 131072" "25 131072" "19 262144" "25 262144" "20 1048576" "26 1048576"; do
    set -- $spec
    timeout 120 python scripts/cluster_timeline.py --variant $1 --n $2 >> $O/ctl.jsonl 2>&1
  done
done
for rep in 1 2 3; do timeout 300 python scripts/sweep.py --logs 17,18 --dtypes i64,f64 >> $O/sweep.jsonl 2>&1; done
