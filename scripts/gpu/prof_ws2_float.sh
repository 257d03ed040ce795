# ncu --set full of the persistent kernel, i32 vs f32 at 2^28 (why f32 sits 3-4 % lower)
for d in i32 f32; do
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:scan_ws2_kernel -s 2 -c 1 \
  -o gpurun_out/prof_ws2_$d python scripts/profile_scan.py --dtype $d > gpurun_out/ncu_ws2_$d.log 2>&1
echo "ncu $d rc=$?"
done
