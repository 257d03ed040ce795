#!/bin/bash
# compile-time word funnel in the shifted-window kernel: GPU suite + misaligned lab (x2)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2ae; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
for rep in 1 2; do timeout 300 python scripts/misaligned_lab.py >> $O/misaligned.log 2>&1; done
cat $O/misaligned.log | grep -v "^$" | tail -8
