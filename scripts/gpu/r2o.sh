#!/bin/bash
# XL cluster geometry with its own cluster size: parity suites + A/B at mid n
cd "$(dirname "$0")/../.."
O=gpurun_out/r2o; mkdir -p $O
timeout 900 python -m pytest tests/test_cluster_gpu.py tests/test_scan_gpu.py tests/test_ops_gpu.py -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
for rep in 1 2 3; do
  timeout 300 python scripts/xl_ab.py >> $O/ab.jsonl 2>&1
  LSCAN_NO_XL=1 timeout 300 python scripts/xl_ab.py >> $O/ab.jsonl 2>&1
done
grep query $O/ab.jsonl | head -2
