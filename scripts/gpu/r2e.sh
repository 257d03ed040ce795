#!/bin/bash
# f64 fast max/min, shifted-window geometry + fast path, reduce kernel
# (256-bit loads, reverse sweep, evict-last head): GPU tests, mode matrix,
# misaligned lab, shard-step pieces, torchrun world 1; look-ahead lab at mid n
cd "$(dirname "$0")/../.."
O=gpurun_out/r2e; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1
timeout 200 python scripts/reduce_lab.py > $O/pieces.json 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 1 --force-dist --steps 20 --warmup 5 --no-sweep --no-sustained > $O/bench_dist1.json 2> $O/bench_dist1.err
for dt in i32 f32; do
  timeout 300 python scripts/lab.py --dtype $dt --op max --shift --cfgs 60,34,40,61 --reps 100 --labso liblscanlab_base.so > $O/shift_max_$dt.json 2>&1
done
for lib in base la1 la2 la3; do
  for lg in 21 22 23 24; do
    timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_$lib.so --graph --reps 200 > $O/la_${lib}_i32_$lg.json 2>&1
    timeout 100 python scripts/lab.py --dtype i64 --n $((1<<(lg-1))) --cfgs 61 --labso liblscanlab_$lib.so --graph --reps 200 > $O/la_${lib}_i64_$((lg-1)).json 2>&1
  done
done
tail -2 $O/gputest.log
