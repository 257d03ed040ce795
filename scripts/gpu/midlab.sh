# persistent-kernel geometries at mid n, graph-timed (device time per call)
for d in i32 i64; do for lg in 20 21 22 23 24; do
timeout 120 python scripts/lab.py --graph --product --dtype $d --n $((1<<lg)) --reps 50 --cfgs 34,40,36,37,46,47,48,49,50,51 2>&1 | tail -1
done; done
