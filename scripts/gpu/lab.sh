# geometry / protocol laboratory runs (one GPU): lab configs, sweep, PCIe, sharded-step pieces, virtual GPUs
set -x
timeout -s KILL 300 python scripts/lab.py --cfgs 30,31,32,34,40,41 > gpurun_out/lab.json 2>&1
timeout -s KILL 300 python scripts/lab.py --wide --cfgs 30,34,40,43 > gpurun_out/lab_wide.json 2>&1
timeout -s KILL 900 python scripts/sweep.py > gpurun_out/sweep.jsonl 2>&1
timeout -s KILL 400 python scripts/pcie_lab.py > gpurun_out/pcie.json 2>&1
timeout -s KILL 300 python scripts/reduce_lab.py > gpurun_out/reduce_lab.json 2>&1
timeout -s KILL 300 python scripts/cyclic_lab.py > gpurun_out/cyclic_lab.json 2>&1
