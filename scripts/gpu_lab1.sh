set -x
timeout -s KILL 300 python scripts/lab.py > gpurun_out/lab1.json 2> gpurun_out/lab1.err
echo "lab rc=$?"
cat gpurun_out/lab1.json; tail -5 gpurun_out/lab1.err
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/bench_ncu.log 2>&1
echo "ncu-launch rc=$?"
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_kernel -s 2 -c 1 -o gpurun_out/prof_r1 python scripts/lab.py --ncu > gpurun_out/ncu_full.log 2>&1
echo "ncu-full rc=$?"
tail -5 gpurun_out/ncu_full.log
