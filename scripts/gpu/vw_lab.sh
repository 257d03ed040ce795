# 32-byte scanner rows (VW = 2) vs the production rows, add and max, 2^28, graph-timed
for op in add max; do
  for d in i32 f32; do timeout 300 python scripts/lab.py --dtype $d --op $op --cfgs 34,60,34,60 --graph --reps 30; done
  for d in i64 f64; do timeout 300 python scripts/lab.py --dtype $d --op $op --cfgs 40,61,40,61 --graph --reps 30; done
done
