#!/bin/bash
# 64-bit max: in-lane prefixes kept in place (pipmm) and + NaN-free f64 scans
# (pipmmnf) against the product build (base), aligned and shifted
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bb; mkdir -p $O
for rep in 1 2; do
  for v in base pipmm pipmmnf; do
    for d in f64 i64; do
      for sh in "" "--shift"; do
        [ $d = i64 ] && [ $v = pipmmnf ] && continue
        echo; echo "== $d max $v $sh rep$rep"
        timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --op max --cfgs 61 --reps 100 $sh 2>&1 | tr -d "\n "
      done
    done
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg61[^}]*}" 
