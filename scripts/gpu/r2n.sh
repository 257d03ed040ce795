#!/bin/bash
# extra-large cluster geometry (16 rows, 64 KiB tiles): cluster/scan parity
# suites, then the 2^19..2^23 sweep with it (default) and without (LSCAN_NO_XL=1)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2n; mkdir -p $O
timeout 900 python -m pytest tests/test_cluster_gpu.py tests/test_scan_gpu.py tests/test_ties_gpu.py tests/test_ops_gpu.py -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
python -c "
from paper_1604_04815_b200 import scan as S; import torch
for dt in (torch.int32, torch.int64, torch.float32, torch.float64): print(dt, S.query_cluster(dt))" > $O/query.txt 2>&1
for rep in 1 2; do
timeout 600 python scripts/sweep.py --min-log 19 --max-log 23 >> $O/sweep_xl.jsonl 2>&1
LSCAN_NO_XL=1 timeout 600 python scripts/sweep.py --min-log 19 --max-log 23 --no-cub >> $O/sweep_noxl.jsonl 2>&1
done
cat $O/query.txt
