#!/bin/bash
# second reducer for add in the aligned kernel (red2add) vs one (small), mid n to 2^28
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ai; mkdir -p $O
for rep in 1 2; do
for lib in small red2add; do
  for lg in 22 23 24 25 26 28; do
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/i32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype f32 --n $((1<<lg)) --cfgs 65 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/f32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype i64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/i64.jsonl 2>&1
  done
done
done
