for cfg in 12 13 17 18 19 20 15; do
  timeout -s KILL 45 python scripts/lab.py --cfgs $cfg --flags 0 --reps 10 > gpurun_out/lab5_$cfg.json 2> gpurun_out/lab5_$cfg.err
  echo "cfg $cfg rc=$?"; grep -A4 '"cfg' gpurun_out/lab5_$cfg.json | tr -d '\n '; echo
done
