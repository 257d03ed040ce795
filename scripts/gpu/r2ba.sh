#!/bin/bash
# f64 max: exact DSETP-pair scans (base) vs NaN-free (a > b) ? a : b scans on
# chunks without NaNs (f64nanfree), aligned and shifted; i64 max beside
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ba; mkdir -p $O
for rep in 1 2; do
  for v in base f64nanfree; do
    for sh in "" "--shift"; do
      echo; echo "== f64 max $v $sh rep$rep"
      timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype f64 --op max --cfgs 61 --reps 100 $sh 2>&1 | tr -d "\n "
    done
  done
  echo; echo "== i64 max base rep$rep"
  timeout 120 python scripts/lab.py --labso liblscanlab_base.so --dtype i64 --op max --cfgs 61 --reps 100 2>&1 | tr -d "\n "
done > $O/ab.log 2>&1
for d in f64 i64; do
  echo; echo "== timing $d max"; timeout 120 python scripts/lab.py --labso liblscanlab_timing.so --dtype $d --op max --cfgs 61 --reps 50 --timing 2>&1 | tr -d "\n "
done > $O/timing.log 2>&1
cat $O/ab.log
cat $O/timing.log
