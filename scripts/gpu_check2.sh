set -x
timeout -s KILL 200 python scripts/lab.py --cfgs 10,12,13,17,18,19,20 --flags 0 > gpurun_out/lab4.json 2> gpurun_out/lab4.err
echo "lab rc=$?"
cat gpurun_out/lab4.json; tail -3 gpurun_out/lab4.err
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu3.log 2>&1
echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu3.log
