#!/bin/bash
# dominating-carry rows for 64-bit max (LS_MAXMIN_DOMINATE 1: f64, 2: + i64)
# against the production-geometry lab build (small), random and ascending data
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bf; mkdir -p $O
run() { # lib dtype data [--shift]
  echo; echo "== $2 max $1 $3 $4"
  timeout 120 python scripts/lab.py --labso liblscanlab_$1.so --dtype $2 --op max --cfgs 61 --reps 100 --data $3 $4 2>&1 | tr -d "\n "
}
for rep in 1 2; do
  for v in small dom1 dom2; do run $v f64 random; run $v f64 random --shift; run $v f64 ascending; done
  for v in small dom2; do run $v i64 random; run $v i64 ascending; done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
