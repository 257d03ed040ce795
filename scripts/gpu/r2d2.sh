#!/bin/bash
# the N>1 code path at world size 1 on the round's last build (torchrun)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2d2; mkdir -p $O
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 \
  bench.py --gpus 1 --force-dist --steps 20 --warmup 5 --no-sweep --no-sustained > $O/bench_dist1.json 2> $O/bench_dist1.err; echo dist=$?
python -c "
import json; a=json.loads(open('$O/bench_dist1.json').readline())
print(a['value'], a.get('validated'), a['config'].get('workload'))
print({k: (a[k].get('value') if isinstance(a[k], dict) else a[k]) for k in ('fused_cyclic','config4','e2e','cpu_baseline') if k in a})
print({k: a['fused_cyclic'].get(k) for k in ('validated','error')} if 'fused_cyclic' in a else None)"
