#!/bin/bash
# latency kernel: early cluster-aggregate publication (remote mbarrier) vs after
# the cluster barrier; cluster parity suites; timelines; product mid-n sweep
cd "$(dirname "$0")/../.."
O=gpurun_out/r2w; mkdir -p $O
timeout 900 python -m pytest tests/test_cluster_gpu.py tests/test_scan_gpu.py tests/test_ops_gpu.py tests/test_ties_gpu.py -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
for rep in 1 2; do
for lib in libclusterlab.so libclusterlab_noearly.so; do
  for spec in "7 524288" "15 2097152" "19 131072" "19 262144" "20 524288" "20 1048576"; do
    set -- $spec
    timeout 120 python scripts/cluster_timeline.py --variant $1 --n $2 --lib $lib >> $O/cl.jsonl 2>&1
  done
done
done
for spec in "15 2097152" "20 1048576"; do set -- $spec; timeout 120 python scripts/cluster_timeline.py --variant $1 --n $2 >> $O/ctl.jsonl 2>&1; done
timeout 600 python scripts/sweep.py --min-log 16 --max-log 22 > $O/sweep.jsonl 2>&1; echo sweep=$?
tail -1 $O/sweep.jsonl
