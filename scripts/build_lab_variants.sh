#!/bin/bash
# Build the persistent-kernel lab library (bench_support/lscan_lab.cu) under the
# compile-time lab switches of lscan_scan_ws2.cuh, as
# bench_support/_build/liblscanlab_<name>.so, for scripts/lab.py --labso,
# scripts/gpu_sustain.sh and scripts/gpu_floatlab.sh.  Runs here (nvcc
# cross-compiles); the .so files travel to the GPU box with the repo.
#   base         product defaults
#   skipred      no reducer pass over the stage      (timing only: wrong sums)
#   skiprow      no row warp scans                   (timing only: wrong sums)
#   skipboth     both of the above                   (timing only)
#   skiplb       no look-back                        (timing only)
#   timing       per-warp-role clock64 totals        (scripts/lab.py --timing)
#   sleep200 / sleep1000   look-back back-off in ns
#   evictnormal  evict-normal L2 policy on the TMA loads
#   nopack       f32 add without the packed FADD2 forms (LS_F32_PACKED=0)
#   f64fast      f64 max/min fast scans on chunks without zeros or NaNs
#   la1/la2/la3  the producer's first ring fill keeps 1/2/3 tile loads in flight
set -e
cd "$(dirname "$0")/.."
declare -A FLAGS=(
  [base]="" [skipred]="-DLS_LAB_SKIP_REDUCE=1" [skiprow]="-DLS_LAB_SKIP_ROWSCAN=1"
  [skipboth]="-DLS_LAB_SKIP_REDUCE=1 -DLS_LAB_SKIP_ROWSCAN=1" [skiplb]="-DLS_LAB_SKIP_LOOKBACK=1"
  [timing]="-DLS_LAB_TIMING=1" [sleep200]="-DLS_LOOKBACK_SLEEP_NS=200" [sleep1000]="-DLS_LOOKBACK_SLEEP_NS=1000"
  [evictnormal]="-DLS_TMA_EVICT_FIRST=0" [nopack]="-DLS_F32_PACKED=0"
  [f64fast]="-DLS_F64_FAST_SCAN=1"
  [la1]="-DLS_LAB_LOOKAHEAD=1" [la2]="-DLS_LAB_LOOKAHEAD=2" [la3]="-DLS_LAB_LOOKAHEAD=3"
)
names=("$@")
[ ${#names[@]} -eq 0 ] && names=("${!FLAGS[@]}")
mkdir -p bench_support/_build
for v in "${names[@]}"; do
  nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -shared ${FLAGS[$v]} \
    -Ipaper_1604_04815_b200/csrc -Iinclude -o bench_support/_build/liblscanlab_$v.so bench_support/lscan_lab.cu &
done
wait
echo "built: ${names[*]}"
