timeout -s KILL 900 python -m pytest tests/test_properties_gpu.py -q -k two_pow_33 > gpurun_out/pytest_2p33.log 2>&1; echo "2p33 test rc=$?"; tail -3 gpurun_out/pytest_2p33.log
timeout -s KILL 600 python bench.py --n 8589934592 --steps 20 --warmup 3 > gpurun_out/bench_2p33.log 2>&1; echo "bench 2p33 rc=$?"; tail -1 gpurun_out/bench_2p33.log | cut -c1-900
