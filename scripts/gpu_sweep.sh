timeout -s KILL 900 python scripts/sweep.py > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
echo "sweep rc=$?"; grep -v sweep gpurun_out/sweep.jsonl | cut -c1-250; tail -3 gpurun_out/sweep.err
