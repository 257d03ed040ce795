#!/bin/bash
# Re-entry check of HEAD (290c79f kernels): smoke, GPU suite, bench N=1,
# reference arm, torchrun world 1, mode matrix, misaligned lab
cd "$(dirname "$0")/../.."
O=gpurun_out/r2f; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=15 > $O/gputest.log 2>&1; echo tests=$?
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 1 --force-dist --steps 10 --warmup 3 > $O/bench_dist1.json 2> $O/bench_dist1.err; echo dist=$?
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1; echo mm=$?
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
tail -3 $O/gputest.log
