timeout -s KILL 300 python scripts/cyclic_lab.py > gpurun_out/cyclic_lab.json 2>&1; echo "lab rc=$?"; cat gpurun_out/cyclic_lab.json | tail -20
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 1 --force-dist --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_dist2.log 2>&1
echo "dist bench rc=$?"; tail -1 gpurun_out/bench_dist2.log | cut -c1-1500
