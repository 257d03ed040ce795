// lscan_lab.cu — tuning laboratory (not part of include/lscan.h): runs the
// hot kernel (add) under alternative compile-time geometries so
// scripts/lab.py can compare them on the device.  Results of the sweeps that
// chose the production geometry: profiles/r1_lab_ws2*.json.
#include <cuda_runtime.h>

#include <cstdint>

#include "lscan.h"
#include "lscan_scan_ws2.cuh"  // -I paper_1604_04815_b200/csrc

using namespace lscan;

namespace {
int g_lab_dtype = 0;  // ls_dtype: 0 i32, 1 i64, 2 f32, 3 f64

int g_lab_op = 0;     // 0 add, 1 max
int g_lab_shift = 0;  // 1: the shifted-window kernel (x misaligned by a whole number of words)
void *g_lab_timeline = nullptr;  // LS_LAB_TIMELINE builds: per-CTA event times (p.xchg)

struct LabK {
    void (*fn)(const ScanParams);
    int threads;
    size_t smem;
};

#ifndef LS_LAB_EXCL
#define LS_LAB_EXCL 0  // 1: exclusive scans (timing only: lab.py checks inclusive results)
#endif
template <typename T, typename OP, int SW, int TILE, int STAGES, int VW, bool SHIFT>
LabK labk() {
    constexpr bool R2 = ws2_red2<T, OP, false, SHIFT>();
    return {&scan_ws2_kernel<T, OP, SW, TILE, STAGES, LS_LAB_EXCL != 0, false, SHIFT, VW>, ws2_threads_x<SW, false, R2>(),
            scan_ws2_smem_bytes<T, SW, TILE, STAGES, SHIFT, R2, lscan::row_transpose<T, OP>()>()};
}

template <typename T, typename OP, int SW, int TILE, int STAGES, int VW>
LabK pick_s() {
    return g_lab_shift ? labk<T, OP, SW, TILE, STAGES, VW, true>() : labk<T, OP, SW, TILE, STAGES, VW, false>();
}

template <typename OP, int SW, int TILE, int STAGES, int VW>
LabK pick() {
    switch (g_lab_dtype) {
    case 1: return pick_s<int64_t, OP, SW, TILE, STAGES, VW>();
    case 2: return pick_s<float, OP, SW, TILE, STAGES, VW>();
    case 3: return pick_s<double, OP, SW, TILE, STAGES, VW>();
    default: return pick_s<int32_t, OP, SW, TILE, STAGES, VW>();
    }
}

template <int SW, int TILE, int STAGES, int VW = 1>
int run_ws(const void *x, void *y, int64_t n, void *ws, cudaStream_t s, int64_t *grid_out) {
    const bool wide = g_lab_dtype == 1 || g_lab_dtype == 3;
    const LabK k = g_lab_op == 1 ? pick<OpMax, SW, TILE, STAGES, VW>() : pick<OpAdd, SW, TILE, STAGES, VW>();
    void (*f)(const ScanParams) = k.fn;
    const size_t smem = k.smem;
    const int threads = k.threads;
    if (cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1;
    int occ = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)f, threads, smem);
    if (occ < 1) return -3;
    const int64_t tile_elems = TILE / (wide ? 8 : 4);
    const int64_t M = (n + tile_elems - 1) / tile_elems;
    int64_t G = (int64_t)occ * sms;
    if (G > M) G = M;
    if (grid_out) *grid_out = G;
    ScanParams p{};
    p.x = x;
    p.y = y;
    p.n = n;
    p.ws = static_cast<uint8_t *>(ws);
    p.num_tiles = M;
    p.corrupt_tile = -1;
    p.stall_tile = -1;
    p.x_shift = g_lab_shift ? (int)((uintptr_t)x & 15u) : 0;
    p.xchg = static_cast<uint8_t *>(g_lab_timeline);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, f, p) == cudaSuccess ? 0 : -2;
}
}  // namespace

#ifndef LS_LAB_SMALL
#define LS_LAB_SMALL 0  // 1: only the production geometries (60, 61, 65) — quick variant builds
#endif

// LS_LAB_TIMELINE builds: the device buffer (grid x kTimelineWords u64) the
// kernel writes its per-CTA event times into; nullptr turns the marks off
extern "C" void ls_lab_set_timeline(void *buf) { g_lab_timeline = buf; }

// flags bits 8..9 select the element type (ls_dtype), bit 10 max, bit 11 the
// shifted-window kernel
extern "C" int ls_lab_run(int cfg, int flags, const void *x, void *y, int64_t n, void *ws, void *stream,
                          int64_t *grid_out) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    g_lab_dtype = (flags >> 8) & 3;
    g_lab_op = (flags >> 10) & 1;
    g_lab_shift = (flags >> 11) & 1;
    switch (cfg) {
    // 32-byte scanner rows (VW = 2) on the production geometries: 32-bit (8, 32 KiB, 6)
    // and 64-bit (12, 48 KiB, 4)
    case 60: return run_ws<8, 32768, 6, 2>(x, y, n, ws, s, grid_out);
    case 61: return run_ws<12, 49152, 4, 2>(x, y, n, ws, s, grid_out);
    // f32 add (12 warps, 48 KiB, 16-byte rows)
    case 65: return run_ws<12, 49152, 4, 1>(x, y, n, ws, s, grid_out);
#if !LS_LAB_SMALL
    // round 2: wider 32-byte-row geometries (64-bit max / min, shifted windows)
    case 62: return run_ws<16, 65536, 3, 2>(x, y, n, ws, s, grid_out);
    case 63: return run_ws<16, 32768, 6, 2>(x, y, n, ws, s, grid_out);
    case 64: return run_ws<16, 49152, 4, 2>(x, y, n, ws, s, grid_out);
    case 30: return run_ws<16, 32768, 4>(x, y, n, ws, s, grid_out);
    case 31: return run_ws<16, 32768, 5>(x, y, n, ws, s, grid_out);
    case 32: return run_ws<16, 32768, 6>(x, y, n, ws, s, grid_out);
    case 33: return run_ws<16, 32768, 7>(x, y, n, ws, s, grid_out);
    case 34: return run_ws<8, 32768, 6>(x, y, n, ws, s, grid_out);
    case 35: return run_ws<16, 65536, 3>(x, y, n, ws, s, grid_out);
    case 36: return run_ws<16, 16384, 12>(x, y, n, ws, s, grid_out);
    case 37: return run_ws<8, 16384, 12>(x, y, n, ws, s, grid_out);
    case 38: return run_ws<24, 49152, 4>(x, y, n, ws, s, grid_out);
    case 40: return run_ws<12, 49152, 4>(x, y, n, ws, s, grid_out);
    case 41: return run_ws<8, 32768, 5>(x, y, n, ws, s, grid_out);
    case 42: return run_ws<8, 32768, 4>(x, y, n, ws, s, grid_out);
    case 43: return run_ws<12, 49152, 3>(x, y, n, ws, s, grid_out);
    case 44: return run_ws<16, 65536, 3>(x, y, n, ws, s, grid_out);
    case 45: return run_ws<4, 32768, 6>(x, y, n, ws, s, grid_out);
    // mid-n candidates: smaller tiles / fewer stages, several CTAs per SM
    case 46: return run_ws<8, 16384, 4>(x, y, n, ws, s, grid_out);
    case 47: return run_ws<4, 16384, 4>(x, y, n, ws, s, grid_out);
    case 48: return run_ws<8, 16384, 3>(x, y, n, ws, s, grid_out);
    case 49: return run_ws<4, 8192, 4>(x, y, n, ws, s, grid_out);
    case 50: return run_ws<8, 32768, 2>(x, y, n, ws, s, grid_out);
    case 51: return run_ws<4, 16384, 2>(x, y, n, ws, s, grid_out);
#endif
    }
    return -3;
}
