#!/bin/bash
# second reducer for 32-bit max / min in the shifted-window kernel (lab A/B)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2t; mkdir -p $O
for rep in 1 2; do
for lib in small shred2_32; do
  for dt in f32 i32; do
    timeout 200 python scripts/lab.py --dtype $dt --op max --shift --cfgs 61 --labso liblscanlab_$lib.so --reps 100 >> $O/shift_max.jsonl 2>&1
  done
done
done
