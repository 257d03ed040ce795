#!/bin/bash
# persistent kernel, i32: predicated-shuffle row scans (wspred) vs C++ form (small), burst + sustained, alternating
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ad; mkdir -p $O
for rep in 1 2; do
for lib in small wspred; do
  timeout 100 python scripts/lab.py --dtype i32 --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/burst.jsonl 2>&1
  timeout 100 python scripts/lab.py --dtype i32 --n $((1<<24)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/burst.jsonl 2>&1
done
done
for lib in small wspred small wspred; do
  timeout 300 python scripts/lab.py --dtype i32 --cfgs 60 --labso liblscanlab_$lib.so --reps 300 --sustain 8 >> $O/sustain.jsonl 2>&1
done
