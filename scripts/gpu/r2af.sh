#!/bin/bash
# contiguous-shard host path simplified: distributed GPU tests + torchrun world-1 bench (e2e)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2af; mkdir -p $O
timeout 600 python -m pytest tests/test_distributed_gpu.py tests/test_bench_gpu.py -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29523 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 --no-sweep --no-sustained > $O/bench_dist1.json 2> $O/bench_dist1.err; echo dist=$?
python -c "
import json; d=json.loads(open('$O/bench_dist1.json').read().strip().splitlines()[-1]); print('value', d['value'], 'e2e', d['e2e'])"
