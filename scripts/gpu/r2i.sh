#!/bin/bash
# mid-n timelines (cyclic vs contiguous deal), ring look-ahead at mid n,
# shifted-window f32 max reducer (misaligned lab + parity suites)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2i; mkdir -p $O
timeout 600 python -m pytest tests/test_ties_gpu.py tests/test_ops_gpu.py tests/test_scan_gpu.py -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
for lg in 20 21 22 23; do
  for c in "" "--contig"; do
    timeout 120 python scripts/timeline_lab.py --dtype i32 --n $((1<<lg)) $c >> $O/timeline.jsonl 2>&1
  done
done
for c in "" "--contig"; do
  timeout 120 python scripts/timeline_lab.py --dtype i64 --n $((1<<21)) $c >> $O/timeline.jsonl 2>&1
  timeout 120 python scripts/timeline_lab.py --dtype f32 --n $((1<<22)) $c >> $O/timeline.jsonl 2>&1
done
for lib in small sla1 sla2 sla3; do
  for lg in 21 22 23 24; do
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 200 >> $O/la_i32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype i64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 200 >> $O/la_i64.jsonl 2>&1
  done
done
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
tail -2 $O/gputest.log
