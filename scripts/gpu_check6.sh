timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu7.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu7.log
timeout -s KILL 600 python scripts/sweep.py --max-log 22 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
echo "sweep rc=$?"; grep -v sweep gpurun_out/sweep2.jsonl | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['dtype'],d['log2n'],d['graph_ms'],d['graph_gelems'],d['cub_gelems'])"
