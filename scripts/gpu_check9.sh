timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu9.log 2>&1
echo "pytest rc=$?"; tail -5 gpurun_out/pytest_gpu9.log
