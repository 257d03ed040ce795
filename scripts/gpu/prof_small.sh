# ncu --set full of the small-n cluster kernel (one block and sixteen blocks)
for lg in 10 18; do
timeout -s KILL 300 ncu --set full --clock-control none --cache-control none --import-source on -k regex:scan_cluster_kernel -s 3 -c 1 \
  -o gpurun_out/prof_cluster_2p$lg python scripts/profile_scan.py --dtype i32 --n $((1<<lg)) --reps 6 > gpurun_out/ncu_cluster_$lg.log 2>&1
echo "ncu $lg rc=$?"
done
