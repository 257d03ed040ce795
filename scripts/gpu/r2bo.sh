#!/bin/bash
# f64 / i64 max exclusive (lab, timing only) with and without in-place
# prefixes; inclusive beside (small, inclpipm); 2 s idle before each run
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bo; mkdir -p $O
for rep in 1 2; do
  for v in small excl exclpipm inclpipm; do
    for d in f64 i64; do
      sleep 2; echo; echo "== $d max $v rep$rep"
      timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --op max --cfgs 61 --reps 100 2>&1 | tr -d "\n "
    done
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
