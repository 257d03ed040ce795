#!/bin/bash
# add: round fold by every CTA (srfold), first-fill look-ahead 1 (sla1), both
# (srfla1) vs the product geometry (small), 2^20 .. 2^28, i32 / i64 / f32
cd "$(dirname "$0")/../.."
O=gpurun_out/r2l; mkdir -p $O
for rep in 1 2; do
for lg in 20 21 22 23 24 25 26 28; do
  for lib in small sla1 srfold srfla1; do
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/i32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype i64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/i64.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype f32 --n $((1<<lg)) --cfgs 65 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/f32.jsonl 2>&1
  done
done
done
