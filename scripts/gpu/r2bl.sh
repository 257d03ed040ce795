#!/bin/bash
# f64 max reducers: order-free max.f64 + NaN screen (f64red) vs exact (small)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bl; mkdir -p $O
for rep in 1 2 3; do
  for v in small f64red; do
    echo; echo "== f64 max $v rep$rep"
    timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype f64 --op max --cfgs 61 --reps 100 2>&1 | tr -d "\n "
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
