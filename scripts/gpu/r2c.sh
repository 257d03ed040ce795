#!/bin/bash
# the session's check of the final build: smoke, GPU suite, bench N=1,
# reference arm, then (each after its own command exited 0 without ncu) the
# bench launch list and ncu --set full of the i32 add and f64 max scans
cd "$(dirname "$0")/../.."
O=gpurun_out/r2c; mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo bench=$?
timeout 300 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; echo ref=$?
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu \
  > $O/bench_ncu.log 2>&1; echo ncu_launches=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 2 -c 1 \
  -o $O/prof_r2c_i32 python scripts/profile_scan.py --dtype i32 > $O/ncu_i32.log 2>&1; echo ncu_i32=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 2 -c 1 \
  -o $O/prof_r2c_f64max python scripts/profile_scan.py --dtype f64 --op max > $O/ncu_f64max.log 2>&1; echo ncu_f64max=$?
