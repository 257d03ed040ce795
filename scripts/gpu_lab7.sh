for w in "" "--wide"; do
for cfg in 39 30 31 32 34 40 41 42; do
  timeout -s KILL 45 python scripts/lab.py $w --cfgs $cfg --flags 0 --reps 30 > gpurun_out/lab7_$cfg$w.json 2> gpurun_out/lab7_$cfg$w.err
  echo "cfg $cfg $w rc=$?"; grep -A4 '"cfg' gpurun_out/lab7_$cfg$w.json | tr -d '\n '; echo; tail -2 gpurun_out/lab7_$cfg$w.err
done; done
