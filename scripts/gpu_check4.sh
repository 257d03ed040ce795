set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu5.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu5.log
timeout -s KILL 400 python scripts/pcie_lab.py > gpurun_out/pcie.json 2>gpurun_out/pcie.err
echo "pcie rc=$?"; cat gpurun_out/pcie.json; tail -3 gpurun_out/pcie.err
timeout -s KILL 400 python bench.py --no-cpu > gpurun_out/bench4.log 2>&1
echo "bench rc=$?"
tail -2 gpurun_out/bench4.log
for d in i64 f64; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 2 -c 1 -o gpurun_out/prof_ws2b_$d python scripts/profile_scan.py --dtype $d > gpurun_out/ncu_full3_$d.log 2>&1
echo "ncu-full $d rc=$?"
done
