#!/bin/bash
# exclusive f64 / i64 max (timing only): per-element exclusive fold (excl) vs the
# inclusive chain stored one element later (exclshift)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bq; mkdir -p $O
for rep in 1 2 3; do
  for v in excl exclshift; do
    for d in f64 i64; do
      sleep 1; echo; echo "== $d max $v rep$rep"
      timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --op max --cfgs 61 --reps 100 2>&1 | tr -d "\n "
    done
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
