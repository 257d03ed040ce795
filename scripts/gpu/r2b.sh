#!/bin/bash
# round 2: f32 add gap vs i32 (geometries, packed FADD2 on/off, per-phase
# cycles, effective clock) and an ncu capture of the mid-n persistent kernel
cd "$(dirname "$0")/../.."
O=gpurun_out/r2b; mkdir -p $O
for dt in f32 i32; do
  timeout 300 python scripts/lab.py --dtype $dt --cfgs 60,34,30,32,40,61,33 --labso liblscanlab_base.so --reps 100 > $O/geo_$dt.json 2>&1
done
timeout 200 python scripts/lab.py --dtype f32 --cfgs 60,34 --labso liblscanlab_nopack.so --reps 100 > $O/nopack_f32.json 2>&1
for dt in f32 i32; do
  timeout 200 python scripts/lab.py --dtype $dt --cfgs 60 --labso liblscanlab_timing.so --timing --reps 50 > $O/timing_$dt.json 2>&1
  timeout 200 python scripts/lab.py --dtype $dt --cfgs 60 --labso liblscanlab_skiprow.so --reps 100 > $O/skiprow_$dt.json 2>&1
  timeout 200 python scripts/lab.py --dtype $dt --cfgs 60 --labso liblscanlab_skipred.so --reps 100 > $O/skipred_$dt.json 2>&1
done
# mid n: the persistent kernel at 2^22 / 2^23 i32 and the cluster kernel at 2^21, graph-timed product
for lg in 20 21 22 23 24; do
  timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_base.so --graph --product --reps 200 > $O/mid_i32_$lg.json 2>&1
  timeout 100 python scripts/lab.py --dtype i32 --n $((1<<lg)) --cfgs 60 --labso liblscanlab_timing.so --timing --reps 50 > $O/midtiming_i32_$lg.json 2>&1
done
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 3 -c 1 \
  -o $O/prof_ws2_i32_2p22 python scripts/profile_scan.py --dtype i32 --n $((1<<22)) --reps 6 > $O/ncu_22.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 3 -c 1 \
  -o $O/prof_ws2_f32_2p28 python scripts/profile_scan.py --dtype f32 --reps 5 > $O/ncu_f32.log 2>&1
timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 3 -c 1 \
  -o $O/prof_ws2_i32_2p28 python scripts/profile_scan.py --dtype i32 --reps 5 > $O/ncu_i32.log 2>&1
ls $O
