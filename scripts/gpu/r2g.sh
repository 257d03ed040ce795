#!/bin/bash
# f64 max/min with the fast scans off (product) vs on (lab f64fast); mid-n
# persistent-kernel phase timing and ncu captures of the mid-n kernels
cd "$(dirname "$0")/../.."
O=gpurun_out/r2g; mkdir -p $O
timeout 400 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1; echo mm=$?
timeout 300 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
for lib in base f64fast; do
  timeout 200 python scripts/lab.py --dtype f64 --op max --cfgs 61,60 --labso liblscanlab_$lib.so --reps 100 > $O/f64max_$lib.json 2>&1
  timeout 200 python scripts/lab.py --dtype f64 --op max --shift --cfgs 61,60 --labso liblscanlab_$lib.so --reps 100 > $O/f64max_shift_$lib.json 2>&1
done
for lg in 20 21 22 23 24; do
  timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_timing.so --timing --reps 50 > $O/midtiming_i32_$lg.json 2>&1
  timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_base.so --graph --product --reps 200 > $O/mid_i32_$lg.json 2>&1
done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 3 -c 1 \
  -o $O/prof_ws2_i32_2p22 python scripts/profile_scan.py --dtype i32 --n $((1<<22)) --reps 6 > $O/ncu_22.log 2>&1; echo ncu22=$?
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:scan_cluster_kernel -s 3 -c 1 \
  -o $O/prof_cluster_i64_2p20 python scripts/profile_scan.py --dtype i64 --n $((1<<20)) --reps 6 > $O/ncu_i64_20.log 2>&1; echo ncu20=$?
ls $O
