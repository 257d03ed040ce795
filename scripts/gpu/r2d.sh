#!/bin/bash
# f32 geometry + shifted-window second reducer: GPU tests, misaligned product
# lab, shifted-window geometry lab, 64-bit max geometry lab
cd "$(dirname "$0")/../.."
O=gpurun_out/r2d; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1
timeout 300 python scripts/mode_matrix.py > $O/mode_matrix.log 2>&1
for dt in i32 f32; do
  timeout 300 python scripts/lab.py --dtype $dt --shift --cfgs 60,34,40,61,63,64 --reps 100 --labso liblscanlab_base.so > $O/shift_add_$dt.json 2>&1
done
for dt in i64 f64; do
  timeout 300 python scripts/lab.py --dtype $dt --shift --cfgs 61,62,63,64,60 --reps 100 --labso liblscanlab_base.so > $O/shift_add_$dt.json 2>&1
  timeout 300 python scripts/lab.py --dtype $dt --op max --shift --cfgs 61,62,63,64,60 --reps 100 --labso liblscanlab_base.so > $O/shift_max_$dt.json 2>&1
  timeout 300 python scripts/lab.py --dtype $dt --op max --cfgs 61,62,63,64,60 --reps 100 --labso liblscanlab_base.so > $O/max_$dt.json 2>&1
done
tail -2 $O/gputest.log
