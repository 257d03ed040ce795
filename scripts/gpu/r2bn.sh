#!/bin/bash
# f64 / i64 rows of the mode matrix back to back and with 2 s idle before
# each row, with the effective SM clock after each row
cd "$(dirname "$0")/../.."
O=gpurun_out/r2bn; mkdir -p $O
MM_DTYPES=i64,f64 timeout 600 python scripts/mode_matrix.py > $O/mm_hot.json 2> $O/mm_hot.err
MM_DTYPES=i64,f64 MM_COOL=2 timeout 600 python scripts/mode_matrix.py > $O/mm_cool.json 2> $O/mm_cool.err
timeout 900 python scripts/mode_matrix.py > $O/mm_all.json 2> $O/mm_all.err
for f in mm_hot mm_cool mm_all; do echo "== $f"; python -c "
import json; d=json.load(open('$O/$f.json'))
for k, v in d.items():
    if isinstance(v, dict) and ('64' in k): print(k, v['gelems'], v['frac_of_measured_hbm'], v['sm_mhz_after'])"; done
