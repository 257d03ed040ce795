timeout -s KILL 600 python -m pytest tests/test_cyclic_gpu.py -x -q > gpurun_out/pytest_cyclic.log 2>&1
echo "cyclic rc=$?"; tail -30 gpurun_out/pytest_cyclic.log
