set -x
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -k "not slow" > gpurun_out/pytest_gpu6.log 2>&1
echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu6.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --force-dist --steps 100 --warmup 5 --no-cpu > gpurun_out/bench_dist1.log 2>&1
echo "dist bench rc=$?"; tail -3 gpurun_out/bench_dist1.log
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/bench_ref2.log 2>&1
echo "ref bench rc=$?"; tail -2 gpurun_out/bench_ref2.log
