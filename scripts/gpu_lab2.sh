set -x
timeout -s KILL 200 python scripts/lab.py --cfgs 10,11,12,13,14,15,16,0 --flags 0 > gpurun_out/lab2.json 2> gpurun_out/lab2.err
echo "lab rc=$?"
cat gpurun_out/lab2.json; tail -5 gpurun_out/lab2.err
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu2.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu2.log
timeout -s KILL 300 python bench.py --steps 200 --warmup 10 --no-cpu > gpurun_out/bench2.log 2>&1
echo "bench rc=$?"
tail -3 gpurun_out/bench2.log
