#!/bin/bash
# which multi-cluster geometry at 2^17..2^21: forced 1 (mid) / 2 (large) / 3 (xl) vs auto
cd "$(dirname "$0")/../.."
O=gpurun_out/r2p; mkdir -p $O
for rep in 1 2; do
  timeout 300 python scripts/xl_ab.py geom >> $O/geom.jsonl 2>&1
  for g in 1 2 3; do LSCAN_CLUSTER_GEOM=$g timeout 300 python scripts/xl_ab.py geom >> $O/geom.jsonl 2>&1; done
done
