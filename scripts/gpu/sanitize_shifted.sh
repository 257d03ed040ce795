# memcheck + racecheck of the shifted-window path, each tensor its own cudaMalloc
export PYTORCH_NO_CUDA_MEMORY_CACHING=1
for tool in memcheck racecheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_case.py shifted > gpurun_out/${tool}_shifted.log 2>&1
  echo "$tool shifted rc=$?"; tail -2 gpurun_out/${tool}_shifted.log
done
