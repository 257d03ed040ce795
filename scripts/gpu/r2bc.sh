#!/bin/bash
# 64-bit max at 2^28: which warp role bounds f64 max — product build (base) vs
# no reducer pass (skipred) vs no row warp scans (skiprow); timing-only builds
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bc; mkdir -p $O
for v in base skipred skiprow; do
  for d in f64 i64; do
    echo; echo "== $d max $v"
    timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --op max --cfgs 61 --reps 100 2>&1 | tr -d "\n "
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg61[^}]*}"
