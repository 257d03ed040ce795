#!/bin/bash
# timelines with look-back detail: base (round chain) vs every-CTA round fold vs look-ahead 1
cd "$(dirname "$0")/../.."
O=gpurun_out/r2k; mkdir -p $O
for rep in 1 2; do
for lib in timeline tlrfold tlla1; do
  for lg in 22 24; do timeout 120 python scripts/timeline_lab.py --dtype i32 --n $((1<<lg)) --labso liblscanlab_$lib.so >> $O/tl_$lib.jsonl 2>&1; done
  timeout 120 python scripts/timeline_lab.py --dtype i64 --n $((1<<21)) --labso liblscanlab_$lib.so >> $O/tl_$lib.jsonl 2>&1
done
done
ls $O
