set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
nproc > gpurun_out/nproc.txt; lscpu | head -20 >> gpurun_out/nproc.txt
timeout -s KILL 180 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
tail -5 gpurun_out/smoke.log
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu.log
timeout -s KILL 300 python bench.py --steps 100 --warmup 5 --no-cpu > gpurun_out/bench.log 2>&1
echo "bench rc=$?"
tail -5 gpurun_out/bench.log
