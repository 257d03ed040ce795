#!/bin/bash
# predicated-shuffle warp scan (SHFL + @p add per level) vs the C++ form:
# GPU parity suites; persistent-kernel lab A/B (small vs nopred) and cluster
# kernel A/B (libclusterlab vs _nopred), alternating, two rounds
cd "$(dirname "$0")/../.."
O=gpurun_out/r2s; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
for rep in 1 2; do
for lib in small nopred; do
  for lg in 22 24 28; do
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ws_i32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype f32 --n $((1<<lg)) --cfgs 65 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ws_f32.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype i64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ws_i64.jsonl 2>&1
    timeout 100 python scripts/lab.py --dtype f64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 100 >> $O/ws_f64.jsonl 2>&1
  done
done
for lib in libclusterlab.so libclusterlab_nopred.so; do
  for spec in "0 65536" "7 524288" "15 2097152" "19 262144" "20 1048576"; do
    set -- $spec
    timeout 120 python scripts/cluster_timeline.py --variant $1 --n $2 --lib $lib >> $O/cl.jsonl 2>&1
  done
done
done
