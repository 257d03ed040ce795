#!/bin/bash
# shifted-window f64 max: exact reducers (small) vs order-free + NaN screen (f64red)
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bp; mkdir -p $O
for rep in 1 2 3; do
  for v in small f64red; do
    for sh in "" "--shift"; do
      sleep 1; echo; echo "== f64 max $v $sh rep$rep"
      timeout 120 python scripts/lab.py --labso liblscanlab_$v.so --dtype f64 --op max --cfgs 61 --reps 100 $sh 2>&1 | tr -d "\n "
    done
  done
done > $O/ab.log 2>&1
cat $O/ab.log | grep -o "== .*\|cfg6[0-9][^}]*}"
timeout 900 python -m pytest tests/test_ties_gpu.py tests/test_ops_gpu.py -m gpu -x -q -p no:cacheprovider > $O/ties.log 2>&1; echo ties=$?; tail -n 2 $O/ties.log
