# TMA load cache policy at L2-resident sizes: evict-first vs evict-normal,
# graph-timed sweep 2^21..2^25 (x + y <= 128 MiB for i32 up to 2^24)
for pol in first normal; do
  LSCAN_L2_POLICY=$pol timeout 600 python scripts/sweep.py --min-log 21 --max-log 25 > gpurun_out/l2_policy_$pol.jsonl 2>&1
done
