#!/bin/bash
# host pipeline: ramped head / tail chunks vs equal chunks (and 16 / 64 MiB chunks); drop-in parity
cd "$(dirname "$0")/../.."
O=gpurun_out/r2y; mkdir -p $O
timeout 900 python -m pytest tests/test_dropin_gpu.py tests/test_ordered_gpu.py -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
for rep in 1 2; do
  timeout 300 python scripts/e2e_lab.py >> $O/e2e.jsonl 2>&1
  LSCAN_HOST_RAMP=0 timeout 300 python scripts/e2e_lab.py >> $O/e2e.jsonl 2>&1
  LSCAN_HOST_CHUNK_MB=16 timeout 300 python scripts/e2e_lab.py >> $O/e2e.jsonl 2>&1
  LSCAN_HOST_CHUNK_MB=64 timeout 300 python scripts/e2e_lab.py >> $O/e2e.jsonl 2>&1
done
cat $O/e2e.jsonl
