#!/bin/bash
# shifted-window kernel: second reducer for 32-bit max / min (product) and
# 64-bit add (lab A/B); parity suites, misaligned lab
cd "$(dirname "$0")/../.."
O=gpurun_out/r2u; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
for rep in 1 2; do
for lib in small shred2add; do
  for dt in i64 f64; do
    timeout 200 python scripts/lab.py --dtype $dt --shift --cfgs 61 --labso liblscanlab_$lib.so --reps 100 >> $O/shift_add.jsonl 2>&1
  done
done
done
