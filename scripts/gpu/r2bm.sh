#!/bin/bash
# f64 max in one process: lab exact reducer (small), lab fast reducer
# (f64red) and the product call (fast reducer on), three times
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bm; mkdir -p $O
for rep in 1 2 3; do
  for v in small f64red; do
    echo; echo "== f64 max $v rep$rep"
    timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype f64 --op max --cfgs 61 --reps 100 --product 2>&1 | tr -d "\n "
  done
done > $O/ab.log 2>&1
timeout 600 python scripts/mode_matrix.py > $O/mode_matrix.json 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}\|product[^}]*}"
python -c "
import json; d=json.load(open('$O/mode_matrix.json'))
print({k: v['frac_of_measured_hbm'] for k, v in d.items() if isinstance(v, dict) and 'float64' in k})"
