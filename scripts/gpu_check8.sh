timeout -s KILL 300 python scripts/reduce_lab.py > gpurun_out/reduce_lab.json 2>&1; echo "reduce rc=$?"; cat gpurun_out/reduce_lab.json
timeout -s KILL 400 python scripts/pcie_lab.py > gpurun_out/pcie2.json 2>gpurun_out/pcie2.err; echo "pcie rc=$?"; python -c "
import json; d=json.load(open('gpurun_out/pcie2.json')); print(d[0]); [print(r) for r in d[1:]]"
