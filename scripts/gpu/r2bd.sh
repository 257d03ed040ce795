#!/bin/bash
# transposed row scans (LS_ROW_TRANSPOSE 1/2/3: f64 max/min, 64-bit max/min,
# everything) against the production-geometry lab build (small), 2^28
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bd; mkdir -p $O
run() { # label lib dtype op cfg [--shift]
  echo; echo "== $3 $4 $1 $6"
  timeout 120 python scripts/lab.py --labso liblscanlab_$2.so --dtype $3 --op $4 --cfgs $5 --reps 100 $6 2>&1 | tr -d "\n "
}
for rep in 1 2; do
  for v in small trs1; do run $v $v f64 max 61; run $v $v f64 max 61 --shift; done
  for v in small trs2; do run $v $v i64 max 61; done
  for v in small trs3; do run $v $v i32 add 60; run $v $v f32 add 65; run $v $v f32 max 61; run $v $v i64 add 61; run $v $v f64 add 61; done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
