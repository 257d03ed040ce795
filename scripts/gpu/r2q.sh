#!/bin/bash
# round-2 final measurement of the committed build: smoke, GPU suite, bench
# (N=1, reference arm, torchrun world 1 both layouts), sweep, mode matrix,
# misaligned lab, ncu launch list + --set full per dtype
cd "$(dirname "$0")/../.."
O=gpurun_out/r2q; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=10 > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 > $O/bench_dist1.json 2> $O/bench_dist1.err; echo dist=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 1 --force-dist --path cyclic --steps 20 --warmup 5 > $O/bench_dist1_cyclic.json 2> $O/bench_dist1_cyclic.err; echo distc=$?
timeout 900 python scripts/sweep.py --min-log 10 --max-log 30 > $O/sweep.jsonl 2>&1; echo sweep=$?
tail -1 $O/sweep.jsonl
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1; echo mm=$?
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
bash scripts/gpu/profile.sh r2 > $O/profile.log 2>&1; echo prof=$?
mv gpurun_out/launches_r2.csv gpurun_out/prof_r2_*.ncu-rep gpurun_out/bench_ncu_r2.log gpurun_out/ncu_r2_*.log $O/ 2>/dev/null
ls $O
