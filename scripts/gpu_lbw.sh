# one vs two look-back warps: per-phase timing (lab timing builds), burst and sustained throughput
for d in i32 i64 f32 f64; do c=34; [ $d = i64 ] || [ $d = f64 ] && c=40
  for v in lb1 lb2; do echo "== $d $v"; timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --cfgs $c --reps 50 --timing 2>&1 | grep -A12 cycles_per_tile | tr -d "\n "; echo; done
done
for d in i32 i64 f32 f64; do c=34; [ $d = i64 ] || [ $d = f64 ] && c=40
  for v in base plain2; do for rep in 1 2; do echo "== burst $d $v"; timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --cfgs $c --reps 100 2>&1 | grep -o '"gelems": [0-9.]*\|"ok": [a-z]*' | tr '\n' ' '; echo; done; done
done
bash scripts/gpu_sustain.sh base plain2
