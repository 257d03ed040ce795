# full round check: tests (incl. slow), smoke, bench, reference arm, sweep
timeout -s KILL 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_full.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_full.log
timeout -s KILL 180 python __graft_entry__.py smoke > gpurun_out/smoke_full.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_full.log
timeout -s KILL 400 python bench.py > gpurun_out/bench_full.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/bench_full.log
timeout -s KILL 400 python bench.py --impl reference > gpurun_out/bench_ref_full.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_full.log
