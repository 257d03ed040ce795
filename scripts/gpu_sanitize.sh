for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_case.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_$tool.log
done
