#!/bin/bash
# final measurement of the round-2 build: bench N=1 (+ reference arm), torchrun
# world 1, sweep, mode matrix, misaligned lab, smoke
cd "$(dirname "$0")/../.."
O=gpurun_out/r2z; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29521 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 > $O/bench_dist1.json 2> $O/bench_dist1.err; echo dist=$?
timeout 900 python scripts/sweep.py --min-log 10 --max-log 30 > $O/sweep.jsonl 2>&1; echo sweep=$?
tail -1 $O/sweep.jsonl
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1; echo mm=$?
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
