# stage costs per dtype at 2^28 (lab builds): base vs variants given as arguments
# (build the variants first: scripts/build_lab_variants.sh)
for d in ${DTYPES:-i32 f32 i64 f64}; do
  c=34; [ $d = i64 ] || [ $d = f64 ] && c=40
  for v in ${@:-base skiprow skipred}; do for rep in 1 2; do echo "== $d $v"; timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype $d --cfgs $c --reps 100 2>&1 | grep -o '"gelems": [0-9.]*\|"ok": [a-z]*' | tr '\n' ' '; echo; done; done
done
