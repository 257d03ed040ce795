timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu8.log 2>&1
echo "pytest rc=$?"; tail -15 gpurun_out/pytest_gpu8.log
timeout -s KILL 300 python bench.py --no-cpu --no-e2e > gpurun_out/bench5.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/bench5.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], {k:(v['gelems'],v['cub_gelems']) for k,v in d['per_dtype'].items()})"
