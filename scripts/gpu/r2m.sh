#!/bin/bash
# product with fill look-ahead 1 + per-CTA round folds (add): GPU suite,
# mode matrix, f32 / i32 / i64 lab A/B against the round-1 look-back (schain),
# bench N=1, sweep
cd "$(dirname "$0")/../.."
O=gpurun_out/r2m; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1; echo mm=$?
for lg in 22 24 26 28; do
  for lib in small schain; do
    timeout 100 python scripts/lab.py --dtype f32 --n $((1<<lg)) --cfgs 65 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ab_f32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype f64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ab_f64.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ab_i32.jsonl 2>&1
  done
done
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 900 python scripts/sweep.py --min-log 10 --max-log 30 > $O/sweep.jsonl 2>&1; echo sweep=$?
tail -1 $O/sweep.jsonl
