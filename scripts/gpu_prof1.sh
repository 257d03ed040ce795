set -x
timeout -s KILL 200 python scripts/lab.py --cfgs 10,11,12,13,15,16 --flags 0 > gpurun_out/lab3.json 2> gpurun_out/lab3.err
echo "lab rc=$?"
cat gpurun_out/lab3.json
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1_ws.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/bench_ncu2.log 2>&1
echo "ncu-launch rc=$?"
for d in i32 i64; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws_kernel -s 2 -c 1 -o gpurun_out/prof_ws_$d python scripts/profile_scan.py --dtype $d > gpurun_out/ncu_full_$d.log 2>&1
echo "ncu-full $d rc=$?"
done
timeout -s KILL 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo "ref rc=$?"; tail -2 gpurun_out/bench_ref.log
