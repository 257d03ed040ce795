// lscan_inst.cuh — builds the DtypeKernels table for one element type
// (included by exactly one lscan_inst_<dtype>.cu each).
#pragma once
#include "lscan_dispatch.h"
#include "lscan_cluster.cuh"
#include "lscan_generic.cuh"
#include "lscan_ordered.cuh"
#include "lscan_scan_ws2.cuh"

namespace lscan {

// scanner row width of the persistent kernel: 32-byte lane chunks (one
// 256-bit store, half the warp scans) for every type and operator
// (profiles/r1_lab_vw.log: f64 add 384 -> 410, f32 max 570 -> 592, i64 add
// +1 %, 32-bit add +-0 burst and +1.3 % under sustained load) but f32 add,
// whose 12-warp geometry keeps 16-byte rows (812 vs 804 Gelem/s,
// profiles/r2_f32_geometry.json)
template <typename T, typename OP>
constexpr int ws2_vw() {
    return (std::is_same<T, float>::value && OP::code == 0) ? 1 : 2;
}

template <typename T, typename OP, bool EXCL>
Launch fast_launch() {
    using C = TypeCfg<T>;
    constexpr bool R2 = ws2_red2<T, OP, false, false>();
    return {&scan_ws2_kernel<T, OP, C::kScanWarps, C::kTileBytes, C::kStages, EXCL, false, false, ws2_vw<T, OP>()>,
            ws2_threads_x<C::kScanWarps, false, R2>(),
            scan_ws2_smem_bytes<T, C::kScanWarps, C::kTileBytes, C::kStages, false, R2, row_transpose<T, OP>()>(), C::kTileBytes, C::kStages};
}

// the shifted-window kernel's rows: 16-byte for 32-bit add (785 vs 733
// Gelem/s i32, profiles/r2_shift_geometry.json), else as the aligned kernel.
// y is (16 * ws2_vw)-byte aligned on this path either way
template <typename T, typename OP>
constexpr int shift_vw() {
    return (sizeof(T) == 4 && OP::code == 0) ? 1 : ws2_vw<T, OP>();
}

template <typename T, typename OP, bool EXCL>
Launch shift_launch() {
    using C = ShiftCfg<T>;
    constexpr bool R2 = ws2_red2<T, OP, false, true>();
    return {&scan_ws2_kernel<T, OP, C::kScanWarps, C::kTileBytes, C::kStages, EXCL, false, true, shift_vw<T, OP>()>,
            ws2_threads_x<C::kScanWarps, false, R2>(),
            scan_ws2_smem_bytes<T, C::kScanWarps, C::kTileBytes, C::kStages, true, R2, row_transpose<T, OP>()>(), C::kTileBytes, C::kStages};
}

template <typename T, typename OP, bool EXCL>
Launch multi_launch() {
    using C = MultiCfg<sizeof(T)>;
    // the fused multi-GPU kernel keeps 16-byte rows for 32-bit types
    // (measured 777 vs 765 Gelem/s at world size 1 with 32-byte rows); 64-bit
    // types take 32-byte rows, which halve the per-row carries a lane keeps
    // live (16-byte rows spilled 12 bytes in the i64 instantiations)
    constexpr int VW = sizeof(T) == 8 ? 2 : 1;
    return {&scan_ws2_kernel<T, OP, C::kScanWarps, C::kTileBytes, C::kStages, EXCL, true, false, VW>,
            ws2_threads<C::kScanWarps, true>(), scan_ws2_smem_bytes<T, C::kScanWarps, C::kTileBytes, C::kStages, false, false, row_transpose<T, OP>()>(),
            C::kTileBytes, C::kStages};
}

template <typename T, typename OP, bool EXCL>
Launch generic_launch() {
    return {&scan_generic_kernel<T, OP, kGenThreads, kGenTileBytes, EXCL>, kGenThreads,
            scan_generic_smem_bytes<T, kGenThreads, kGenTileBytes>(), kGenTileBytes, 1};
}

template <typename T, typename OP, bool EXCL, int V, int MINB>
Launch cluster_launch() {
    // 64-bit types in the mid / large geometries: 32-byte lane rows (256-bit
    // accesses, half the warp scans; -5-6 % per call at 2^18-2^20,
    // profiles/r1_cluster_lab_vw.log); 32-bit and the small geometry: neutral
    // or slower, 16-byte rows
    // (the extra-large 16-row geometry takes them for every type: 16-byte rows
    // keep 16 row prefixes live and the 32-bit exclusive forms spilled)
    constexpr int VW = ((sizeof(T) == 8 && V >= 8) || V >= 16) ? 2 : 1;
    return {&scan_cluster_kernel<T, OP, EXCL, V, kClusterThreads, MINB, VW>, kClusterThreads, 0,
            kClusterThreads * V * 16, 1};
}

template <typename T, typename OP>
void fill_op(DtypeKernels &k) {
    k.cluster[OP::code][0][0] = cluster_launch<T, OP, false, kClusterRowsSmall, kClusterMinBlocksSmall>();
    k.cluster[OP::code][1][0] = cluster_launch<T, OP, true, kClusterRowsSmall, kClusterMinBlocksSmall>();
    k.cluster[OP::code][0][1] = cluster_launch<T, OP, false, kClusterRowsMid, kClusterMinBlocksMid>();
    k.cluster[OP::code][1][1] = cluster_launch<T, OP, true, kClusterRowsMid, kClusterMinBlocksMid>();
    k.cluster[OP::code][0][2] = cluster_launch<T, OP, false, kClusterRowsLarge, kClusterMinBlocksLarge>();
    k.cluster[OP::code][1][2] = cluster_launch<T, OP, true, kClusterRowsLarge, kClusterMinBlocksLarge>();
    k.cluster[OP::code][0][3] = cluster_launch<T, OP, false, kClusterRowsXL, kClusterMinBlocksXL>();
    k.cluster[OP::code][1][3] = cluster_launch<T, OP, true, kClusterRowsXL, kClusterMinBlocksXL>();
    k.scan[OP::code][0][1] = fast_launch<T, OP, false>();
    k.scan[OP::code][1][1] = fast_launch<T, OP, true>();
    k.scan[OP::code][0][0] = generic_launch<T, OP, false>();
    k.scan[OP::code][1][0] = generic_launch<T, OP, true>();
    k.multi[OP::code][0] = multi_launch<T, OP, false>();
    k.multi[OP::code][1] = multi_launch<T, OP, true>();
    k.ws2_vw[OP::code] = ws2_vw<T, OP>();
    k.shift[OP::code][0] = shift_launch<T, OP, false>();
    k.shift[OP::code][1] = shift_launch<T, OP, true>();
    k.reduce_fn[OP::code] = (const void *)&reduce_kernel<T, OP, kReduceThreads>;
    k.ordered[OP::code][0] = {&scan_ordered_kernel<T, OP, false>, kOrdThreads, kOrdSmemBytes, kOrdStageBytes, kOrdStages};
    k.ordered[OP::code][1] = {&scan_ordered_kernel<T, OP, true>, kOrdThreads, kOrdSmemBytes, kOrdStageBytes, kOrdStages};
}

template <typename T>
void launch_reduce_t(int op, const void *x, int64_t n, void *total_out, void *ws, int grid, int64_t keep,
                     cudaStream_t s) {
    const T *xp = static_cast<const T *>(x);
    T *tp = static_cast<T *>(total_out);
    uint8_t *w = static_cast<uint8_t *>(ws);
    if (op == OpMax::code) reduce_kernel<T, OpMax, kReduceThreads><<<grid, kReduceThreads, 0, s>>>(xp, n, tp, w, keep);
    else if (op == OpMin::code)
        reduce_kernel<T, OpMin, kReduceThreads><<<grid, kReduceThreads, 0, s>>>(xp, n, tp, w, keep);
    else reduce_kernel<T, OpAdd, kReduceThreads><<<grid, kReduceThreads, 0, s>>>(xp, n, tp, w, keep);
    if constexpr (order_sensitive<T, OpMax>()) {
        // float max/min: the tie fix-up behind it (every block returns at
        // once unless the total is a zero or a NaN)
        if (op == OpMax::code)
            reduce_ties_kernel<T, OpMax, kReduceThreads><<<grid, kReduceThreads, 0, s>>>(xp, n, tp, w);
        else if (op == OpMin::code)
            reduce_ties_kernel<T, OpMin, kReduceThreads><<<grid, kReduceThreads, 0, s>>>(xp, n, tp, w);
    }
}

template <typename T>
void launch_carry_t(int op, const void *totals, int64_t rank, void *carry_out, cudaStream_t s) {
    const T *tp = static_cast<const T *>(totals);
    T *cp = static_cast<T *>(carry_out);
    if (op == OpMax::code) carry_kernel<T, OpMax><<<1, 32, 0, s>>>(tp, rank, cp);
    else if (op == OpMin::code) carry_kernel<T, OpMin><<<1, 32, 0, s>>>(tp, rank, cp);
    else carry_kernel<T, OpAdd><<<1, 32, 0, s>>>(tp, rank, cp);
}

template <typename T>
void launch_stress_t(uint64_t *slots, int64_t count, uint32_t tag, int *writer_done, unsigned long long *stats,
                     int readers, cudaStream_t s) {
    slot_stress_kernel<T><<<1 + readers, 128, 0, s>>>(slots, count, tag, writer_done, stats);
}

template <typename T>
DtypeKernels make_kernels() {
    DtypeKernels k{};
    fill_op<T, OpAdd>(k);
    fill_op<T, OpMax>(k);
    fill_op<T, OpMin>(k);
    k.launch_reduce = &launch_reduce_t<T>;
    k.launch_carry = &launch_carry_t<T>;
    k.launch_stress = &launch_stress_t<T>;
    return k;
}

}  // namespace lscan
