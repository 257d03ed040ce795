# alignment paths after the one-launch dispatch: tests, sanitizer, throughput
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_case.py shifted > gpurun_out/${tool}_shifted.log 2>&1
  echo "$tool shifted rc=$?"; tail -1 gpurun_out/${tool}_shifted.log
done
unset PYTORCH_NO_CUDA_MEMORY_CACHING
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python scripts/misaligned_lab.py > gpurun_out/misaligned_lab.log 2>&1; tail -4 gpurun_out/misaligned_lab.log
