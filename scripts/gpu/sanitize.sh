for mode in full partial generic reduce cluster shifted; do
  timeout -s KILL 600 compute-sanitizer --tool racecheck --print-limit 5 python scripts/sanitize_case.py $mode > gpurun_out/racecheck_$mode.log 2>&1
  echo "racecheck $mode rc=$?"; tail -2 gpurun_out/racecheck_$mode.log
done
for tool in memcheck synccheck initcheck; do
  timeout -s KILL 600 compute-sanitizer --tool $tool --print-limit 10 python scripts/sanitize_case.py all > gpurun_out/sanitize2_$tool.log 2>&1
  echo "$tool rc=$?"; tail -2 gpurun_out/sanitize2_$tool.log
done
timeout -s KILL 600 python -m pytest tests/test_cli.py -q > gpurun_out/pytest_cli.log 2>&1; echo "cli rc=$?"; tail -3 gpurun_out/pytest_cli.log
