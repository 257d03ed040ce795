for i in 1 2 3; do
  timeout -s KILL 900 python -m pytest tests -m gpu -q -x -p no:randomly > gpurun_out/pytest_rep$i.log 2>&1
  echo "rep $i rc=$?"; tail -1 gpurun_out/pytest_rep$i.log
done
