#!/bin/bash
# mbarrier waits with a suspend-time hint (susp) vs spinning try_wait (small):
# burst at 2^22 / 2^24 / 2^28 and 6 blocks of sustained load at 2^28
cd "$(dirname "$0")/../.."
O=gpurun_out/r2v; mkdir -p $O
for rep in 1 2; do
for lib in small susp; do
  for lg in 22 24 28; do
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/i32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype f32 --n $((1<<lg)) --cfgs 65 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/f32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype i64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/i64.jsonl 2>&1
  done
done
done
for lib in small susp; do
  timeout 300 python scripts/lab.py --dtype i32 --cfgs 60 --labso liblscanlab_$lib.so --reps 300 --sustain 6 >> $O/sustain.jsonl 2>&1
done
