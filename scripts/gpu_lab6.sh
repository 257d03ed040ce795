for cfg in 10 17 30 31 32 33 34 35 36 37 38; do
  timeout -s KILL 45 python scripts/lab.py --cfgs $cfg --flags 0 --reps 30 > gpurun_out/lab6_$cfg.json 2> gpurun_out/lab6_$cfg.err
  echo "cfg $cfg rc=$?"; grep -A4 '"cfg' gpurun_out/lab6_$cfg.json | tr -d '\n '; echo; tail -2 gpurun_out/lab6_$cfg.err
done
