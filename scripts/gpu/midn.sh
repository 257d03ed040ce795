for lg in 20 22 24 26; do
  n=$((1<<lg))
  timeout -s KILL 120 python scripts/lab.py --n $n --cfgs 34,32,31,45 --reps 200 > gpurun_out/midn_$lg.json 2>&1; echo "n=2^$lg"; grep -A1 '"cfg' gpurun_out/midn_$lg.json | grep -v "^--" | tr -d '\n '; echo
done
