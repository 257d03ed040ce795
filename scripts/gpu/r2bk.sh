#!/bin/bash
# f64 max geometry with transposed row scans (full lab build 'base'):
# scanner warps / tile / stages / row width, 2^28, twice
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bk; mkdir -p $O
for rep in 1 2; do
  for sh in "" "--shift"; do
    echo; echo "== f64 max $sh rep$rep"
    timeout 300 python scripts/lab.py --labso liblscanlab_base.so --dtype f64 --op max --cfgs 61,62,63,64,40,38 --reps 100 $sh 2>&1 | tr -d "\n "
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg[0-9]*_[^}]*}"
