#!/bin/bash
# product build with transposed row scans for f64 max/min (LS_ROW_TRANSPOSE=1):
# GPU suite, mode matrix at 2^28, misaligned lab
cd "$(dirname "$0")/../.."
O=gpurun_out/r2be; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo tests=$?
tail -2 $O/gputest.log
timeout 600 python scripts/mode_matrix.py > $O/mode_matrix.json 2> $O/mode_matrix.err; echo mm=$?
timeout 600 python scripts/misaligned_lab.py > $O/misaligned.log 2>&1; echo mis=$?
python - <<'PY'
import json
d=json.load(open("gpurun_out/r2be/mode_matrix.json"))
print({k: v["frac_of_measured_hbm"] for k, v in d.items() if isinstance(v, dict) and "float64" in k})
PY
tail -30 $O/misaligned.log
