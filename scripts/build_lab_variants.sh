#!/bin/bash
# Build the persistent-kernel lab library (bench_support/lscan_lab.cu) under the
# compile-time lab switches of lscan_scan_ws2.cuh, as
# bench_support/_build/liblscanlab_<name>.so, for scripts/lab.py --labso,
# scripts/gpu/sustain.sh and scripts/gpu/floatlab.sh.  Runs here (nvcc
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
#   f64nanfree   f64 max/min (a > b) ? a : b scans on chunks without NaNs
#   trs1/2/3     transposed row scans (LS_ROW_TRANSPOSE) for f64 max/min / 64-bit max/min / everything
#   f64red       f64 max/min reducers: order-free max.f64 + f32-view NaN screen (LS_F64_FAST_REDUCE)
#   excl / exclpipm / inclpipm   exclusive scans (timing only) without / with in-place
#                prefixes (LS_PIP_MAXMIN), inclusive with them
#   pipmm        64-bit max/min keep in-lane prefixes in place (LS_PIP_MAXMIN)
#   pipmmnf      pipmm + f64nanfree
#   timeline     per-CTA event times (LS_LAB_TIMELINE; production geometries only)
#   small        production geometries only (cfgs 60, 61, 65)
#   sla1/2/3     small + look-ahead 1/2/3
#   la1/la2/la3  the producer's first ring fill keeps 1/2/3 tile loads in flight (product: 1)
#   schain       small + the round-1 look-back (round chain through CTA G-1, whole first fill at once)
set -e
cd "$(dirname "$0")/.."
declare -A FLAGS=(
  [base]="" [skipred]="-DLS_LAB_SKIP_REDUCE=1" [skiprow]="-DLS_LAB_SKIP_ROWSCAN=1"
  [skipboth]="-DLS_LAB_SKIP_REDUCE=1 -DLS_LAB_SKIP_ROWSCAN=1" [skiplb]="-DLS_LAB_SKIP_LOOKBACK=1"
  [timing]="-DLS_LAB_TIMING=1" [sleep200]="-DLS_LOOKBACK_SLEEP_NS=200" [sleep1000]="-DLS_LOOKBACK_SLEEP_NS=1000"
  [evictnormal]="-DLS_TMA_EVICT_FIRST=0" [nopack]="-DLS_F32_PACKED=0"
  [f64fast]="-DLS_F64_FAST_SCAN=1" [f64nanfree]="-DLS_F64_NANFREE_SCAN=1"
  [trs1]="-DLS_LAB_SMALL=1 -DLS_ROW_TRANSPOSE=1" [trs2]="-DLS_LAB_SMALL=1 -DLS_ROW_TRANSPOSE=2"
  [trs3]="-DLS_LAB_SMALL=1 -DLS_ROW_TRANSPOSE=3"
  [f64red]="-DLS_LAB_SMALL=1 -DLS_F64_FAST_REDUCE=1"
  [excl]="-DLS_LAB_SMALL=1 -DLS_LAB_EXCL=1" [exclpipm]="-DLS_LAB_SMALL=1 -DLS_LAB_EXCL=1 -DLS_PIP_MAXMIN=1"
  [inclpipm]="-DLS_LAB_SMALL=1 -DLS_PIP_MAXMIN=1"
  [pipmm]="-DLS_PIP_MAXMIN=1" [pipmmnf]="-DLS_PIP_MAXMIN=1 -DLS_F64_NANFREE_SCAN=1"
  [timeline]="-DLS_LAB_SMALL=1 -DLS_LAB_TIMELINE=1" [small]="-DLS_LAB_SMALL=1"
  [tlrfold]="-DLS_LAB_SMALL=1 -DLS_LAB_TIMELINE=1 -DLS_ROUND_FOLD=1" [tlla1]="-DLS_LAB_SMALL=1 -DLS_LAB_TIMELINE=1 -DLS_FILL_LOOKAHEAD=1"
  [sla1]="-DLS_LAB_SMALL=1 -DLS_FILL_LOOKAHEAD=1" [sla2]="-DLS_LAB_SMALL=1 -DLS_FILL_LOOKAHEAD=2"
  [sla3]="-DLS_LAB_SMALL=1 -DLS_FILL_LOOKAHEAD=3" [srfold]="-DLS_LAB_SMALL=1 -DLS_ROUND_FOLD=1"
  [nopred]="-DLS_LAB_SMALL=1 -DLS_SHFL_PRED_SCAN=0"
  [shred2_32]="-DLS_LAB_SMALL=1 -DLS_SHIFT_RED2_32=1"
  [shred2add]="-DLS_LAB_SMALL=1 -DLS_SHIFT_RED2_ADD=1"
  [susp]="-DLS_LAB_SMALL=1 -DLS_MBAR_SUSPEND_NS=1000000"
  [wspred]="-DLS_LAB_SMALL=1 -DLS_WS2_PRED_SCAN=1"
  [shnan]="-DLS_LAB_SMALL=1 -DLS_SHIFT_NAN_REDUCE=1 -DLS_SHIFT_RED2_32=0"
  [red2add]="-DLS_LAB_SMALL=1 -DLS_RED2_ADD=1"
  [srfla1]="-DLS_LAB_SMALL=1 -DLS_ROUND_FOLD=1 -DLS_FILL_LOOKAHEAD=1"
  [la1]="-DLS_FILL_LOOKAHEAD=1" [la2]="-DLS_FILL_LOOKAHEAD=2" [la3]="-DLS_FILL_LOOKAHEAD=3"
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
