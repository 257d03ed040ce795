#!/bin/bash
# late in-lane prefixes for 64-bit max (LS_PIP_LATE; pipl: f64, pipl2: + i64
# with transposed row scans) against the production-geometry lab build (small)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bg; mkdir -p $O
run() { # lib dtype [--shift]
  echo; echo "== $2 max $1 $3"
  timeout 120 python scripts/lab.py --labso liblscanlab_$1.so --dtype $2 --op max --cfgs 61 --reps 100 $3 2>&1 | tr -d "\n "
}
for rep in 1 2; do
  for v in small pipl pipl2; do run $v f64; run $v f64 --shift; done
  for v in small pipl2; do run $v i64; run $v i64 --shift; done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
