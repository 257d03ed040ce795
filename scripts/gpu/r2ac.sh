#!/bin/bash
# producer back-off (nanosleep between free-stage polls) vs spinning: burst and sustained
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ac; mkdir -p $O
for rep in 1 2; do
for lib in small pb100 pb400; do
  timeout 100 python scripts/lab.py --dtype i32 --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/burst.jsonl 2>&1
  timeout 100 python scripts/lab.py --dtype f32 --cfgs 65 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/burst.jsonl 2>&1
  timeout 100 python scripts/lab.py --dtype i64 --n $((1<<27)) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/burst.jsonl 2>&1
  timeout 100 python scripts/lab.py --dtype i32 --n $((1<<24)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/burst.jsonl 2>&1
done
done
for lib in small pb100 pb400 small; do
  timeout 300 python scripts/lab.py --dtype i32 --cfgs 60 --labso liblscanlab_$lib.so --reps 300 --sustain 6 >> $O/sustain.jsonl 2>&1
done
