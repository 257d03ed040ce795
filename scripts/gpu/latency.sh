# small/mid-n evidence (BASELINE config 4): latency-kernel tests, host and
# device cost per call, the 2^10..2^24 sweep against CUB (events and graphs)
timeout 900 python -m pytest tests/test_cluster_gpu.py tests/test_scan_gpu.py -x -q > gpurun_out/pytest_latency.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/pytest_latency.log
timeout 300 bench_support/_build/launch_floor > gpurun_out/launch_floor.json 2> gpurun_out/launch_floor.log; echo "floor rc=$?"
timeout 300 python scripts/overhead_lab.py 10 12 14 16 17 18 20 > gpurun_out/overhead.log 2>&1; echo "overhead rc=$?"
timeout 300 python scripts/cluster_lab.py > gpurun_out/cluster_lab.log 2>&1; echo "cluster lab rc=$?"
timeout 900 python scripts/sweep.py --max-log 24 > gpurun_out/sweep_latency.jsonl 2>&1; echo "sweep rc=$?"
