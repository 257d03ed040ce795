set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider --durations=25 > gpurun_out/r2a_gputest.log 2>&1; echo tests=$?
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo bench=$?
timeout 300 python bench.py --impl reference > gpurun_out/r2a_bench_ref.json 2> gpurun_out/r2a_bench_ref.err; echo ref=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --force-dist --steps 10 --warmup 3 > gpurun_out/r2a_bench_dist1.json 2> gpurun_out/r2a_bench_dist1.err; echo dist=$?
tail -3 gpurun_out/r2a_gputest.log
