set -x
free -g | head -2
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu4.log 2>&1
echo "pytest rc=$?"
tail -20 gpurun_out/pytest_gpu4.log
timeout -s KILL 180 python __graft_entry__.py smoke > gpurun_out/smoke2.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/smoke2.log
timeout -s KILL 400 python bench.py > gpurun_out/bench3.log 2>&1
echo "bench rc=$?"
tail -3 gpurun_out/bench3.log
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1_ws2.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/bench_ncu3.log 2>&1
echo "ncu-launch rc=$?"
for d in i32 i64 f32 f64; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 2 -c 1 -o gpurun_out/prof_ws2_$d python scripts/profile_scan.py --dtype $d > gpurun_out/ncu_full2_$d.log 2>&1
echo "ncu-full $d rc=$?"
done
