#!/bin/bash
# shifted windows (x misaligned): transposed row scans for every op (trs3) and
# 64-bit max/min (trs2) against the production-geometry lab build (small)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bh; mkdir -p $O
run() { # lib dtype op cfg
  echo; echo "== $2 $3 $1 shift"
  timeout 120 python scripts/lab.py --labso liblscanlab_$1.so --dtype $2 --op $3 --cfgs $4 --reps 100 --shift 2>&1 | tr -d "\n "
}
for rep in 1 2; do
  for v in small trs3; do run $v f32 max 61; run $v i32 max 61; run $v f32 add 65; done
  for v in small trs2; do run $v i64 max 61; done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
