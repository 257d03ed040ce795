# ncu evidence for the hot kernel (run under gpurun; one GPU; never multi-rank):
#   1. the launch list of a short bench run (per-launch device time, cold/serialised)
#   2. one --set full capture per dtype of the production scan kernel
set -x
tag=${1:-r1}
timeout -s KILL 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-e2e --no-cpu \
  > gpurun_out/bench_ncu_${tag}.log 2>&1
for d in i32 i64 f32 f64; do
  timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 2 -c 1 \
    -o gpurun_out/prof_${tag}_$d python scripts/profile_scan.py --dtype $d > gpurun_out/ncu_${tag}_$d.log 2>&1
done
