# ncu --set full of the latency kernel's mid geometry, i32 2^17 vs i64 2^16 (same bytes, one cluster)
for spec in "i32 17" "i64 16" "i64 15"; do set -- $spec
timeout -s KILL 300 ncu --set full --clock-control none --import-source on --warp-sampling-interval 0 -k regex:scan_cluster_kernel -s 3 -c 1 \
  -o gpurun_out/prof_mid_$1_2p$2 python scripts/profile_scan.py --dtype $1 --n $((1<<$2)) --reps 6 > gpurun_out/ncu_mid_$1_$2.log 2>&1
echo "ncu $1 $2 rc=$?"
done
