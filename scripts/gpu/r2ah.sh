#!/bin/bash
# shifted f32 max: FMNMX3.NAN single reducer (shnan) vs two exact reducers (small), after the compile-time funnel
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ah; mkdir -p $O
for rep in 1 2; do for lib in small shnan; do
  timeout 200 python scripts/lab.py --dtype f32 --op max --shift --cfgs 61 --labso liblscanlab_$lib.so --reps 100 >> $O/ab.jsonl 2>&1
done; done
grep -h -A1 '"cfg61' $O/ab.jsonl
