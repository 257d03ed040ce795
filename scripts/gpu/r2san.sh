#!/bin/bash
# compute-sanitizer on the round-2 build: racecheck per path, memcheck /
# synccheck / initcheck over every case (XL cluster geometry, shifted 32-bit
# max second reducer, per-CTA round folds and fill look-ahead included)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2san; mkdir -p $O
for mode in full partial cluster shifted; do
  timeout -s KILL 900 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_case.py $mode > $O/racecheck_$mode.log 2>&1
  echo "racecheck $mode rc=$?"; tail -2 $O/racecheck_$mode.log
done
for tool in memcheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_case.py all > $O/$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 $O/$tool.log
done
