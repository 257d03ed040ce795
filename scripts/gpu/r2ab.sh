#!/bin/bash
# f64 latency kernel with U[-1,1] data vs integer-valued data; i64 full-range vs small ints
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ab; mkdir -p $O
for rep in 1 2; do
  for d in int unit; do
    for n in 131072 262144; do timeout 120 python scripts/cluster_timeline.py --variant 25 --n $n --data $d --lib libclusterlab.so >> $O/ab.jsonl 2>&1; done
  done
  for d in int fullint; do
    for n in 131072 262144; do timeout 120 python scripts/cluster_timeline.py --variant 19 --n $n --data $d --lib libclusterlab.so >> $O/ab.jsonl 2>&1; done
  done
done
cat $O/ab.jsonl
