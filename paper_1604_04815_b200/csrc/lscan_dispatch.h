// lscan_dispatch.h — internal: per-dtype kernel tables built in the
// lscan_inst_*.cu translation units (compiled in parallel) and consumed by
// lscan_api.cu.  Not part of the public ABI.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "lscan_common.cuh"

namespace lscan {

// ---- geometry (chosen from the lab sweeps) --------------
template <int ES>
struct FastCfg;
// 32-bit elements: 8 scanner warps, 32 KiB tiles (8192 elements), 6 stages
template <>
struct FastCfg<4> {
    static constexpr int kScanWarps = 8, kTileBytes = 32768, kStages = 6;
};
// 64-bit elements: 12 scanner warps, 48 KiB tiles (6144 elements), 4 stages
template <>
struct FastCfg<8> {
    static constexpr int kScanWarps = 12, kTileBytes = 49152, kStages = 4;
};
// per element type: f32 takes the 64-bit geometry — 12 scanner warps hide
// the FADD / FSETP latency chains 8 warps do not (profiles/r2_f32_geometry.json:
// f32 add 792 -> 812 Gelem/s, f32 max 760 -> 814 at 2^28; i32 stays on 8 warps,
// where 12 measure 809 -> 795)
template <typename T>
struct TypeCfg : FastCfg<sizeof(T)> {};
template <>
struct TypeCfg<float> : FastCfg<8> {};
// the shifted-window kernel (x misaligned): 12 scanner warps / 48 KiB for
// every type — the word funnel adds scanner work (profiles/r2_shift_geometry.json:
// i32 add 741 -> 786 Gelem/s with x one element off)
template <typename T>
struct ShiftCfg : FastCfg<8> {};
// the multi-GPU variant carries two more warps (pusher, global chain); the
// 64-bit single-GPU geometry would then spill (17 warps leave ~100
// registers a thread), so 64-bit multi-GPU scans use the 32-bit geometry's
// 8 scanner warps and 32 KiB tiles (ls_query_multi_config reports them: the
// block-cyclic layout follows the tile)
template <int ES>
struct MultiCfg : FastCfg<ES> {};
template <>
struct MultiCfg<8> : FastCfg<4> {};
constexpr int kGenThreads = 512;  // generic (unaligned) path
constexpr int kGenTileBytes = 32768;
constexpr int kReduceThreads = 512;
constexpr int kNumOps = 3;  // ls_op: add, max, min

struct Launch {
    void (*fn)(const ScanParams);
    int threads;
    size_t smem;
    int tile_bytes;
    int stages;
};

struct DtypeKernels {
    Launch scan[kNumOps][2][2];  // [op][exclusive][fast]
    Launch multi[kNumOps][2];    // [op][exclusive]: block-cyclic multi-GPU variant of the fast kernel
    int ws2_vw[kNumOps];         // the persistent kernel's scanner row width in vectors (y alignment 16 * vw)
    Launch shift[kNumOps][2];    // [op][exclusive]: x 16 bytes misaligned, y aligned (shifted TMA window)
    Launch cluster[kNumOps][2][kClusterGeoms];  // [op][exclusive][small, mid, large, xl]: latency kernel (any alignment)
    Launch ordered[kNumOps][2];  // [op][exclusive]: strict left fold, one CTA (the reference's B = 1 path)
    const void *reduce_fn[kNumOps];
    void (*launch_reduce)(int op, const void *x, int64_t n, void *total_out, void *ws, int grid, int64_t keep_bytes,
                          cudaStream_t s);
    void (*launch_carry)(int op, const void *totals, int64_t rank, void *carry_out, cudaStream_t s);
    void (*launch_stress)(uint64_t *slots, int64_t count, uint32_t tag, int *writer_done, unsigned long long *stats,
                          int readers, cudaStream_t s);
};

const DtypeKernels &kernels_i32();
const DtypeKernels &kernels_i64();
const DtypeKernels &kernels_f32();
const DtypeKernels &kernels_f64();

}  // namespace lscan
