// lscan_lab.cu — tuning laboratory (not part of include/lscan.h): runs the
// i32 inclusive TMA scan kernel under alternative compile-time geometries and
// experiment flags so bench/tune scripts can compare them on the device.
#include <cuda_runtime.h>

#include <cstdint>

#include "lscan.h"
#include "lscan_kernels.cuh"
#include "lscan_scan_ws.cuh"
#include "lscan_scan_ws2.cuh"

using namespace lscan;

namespace {
template <int THREADS, int TILE, int STAGES>
int run(int flags, const void *x, void *y, int64_t n, void *ws, cudaStream_t s, int64_t *grid_out) {
    auto f = &scan_kernel<uint32_t, THREADS, TILE, STAGES, false, true>;
    const size_t smem = (size_t)STAGES * TILE + STAGES * 8 + (2 * (THREADS / 32) + 1) * 4 + 16;
    if (cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1;
    int occ = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)f, THREADS, smem);
    const int64_t tile_elems = TILE / 4;
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
    p.experiment = flags;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, f, p) == cudaSuccess ? 0 : -2;
}
int g_lab_dtype = 0;  // 0 = u32, 1 = u64

template <int SW, int TILE, int STAGES, int KIND = 1>
int run_ws(int flags, const void *x, void *y, int64_t n, void *ws, cudaStream_t s, int64_t *grid_out) {
    void (*f)(const ScanParams);
    const bool wide = g_lab_dtype == 1;
    if constexpr (KIND == 1) f = wide ? &scan_ws_kernel<uint64_t, SW, TILE, STAGES, false>
                                      : &scan_ws_kernel<uint32_t, SW, TILE, STAGES, false>;
    else f = wide ? &scan_ws2_kernel<uint64_t, SW, TILE, STAGES, false>
                  : &scan_ws2_kernel<uint32_t, SW, TILE, STAGES, false>;
    const size_t smem = scan_ws_smem_bytes<uint64_t, SW, TILE, STAGES>();
    const int threads = (SW + 3) * 32;
    if (cudaFuncSetAttribute((const void *)f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return -1;
    int occ = 0, dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)f, threads, smem);
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
    p.experiment = flags;
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

extern "C" int ls_lab_run(int cfg, int flags, const void *x, void *y, int64_t n, void *ws, void *stream,
                          int64_t *grid_out) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    g_lab_dtype = (flags >> 8) & 1;  // bit 8 selects 64-bit elements (ws/ws2 configs only)
    flags &= 0xff;
    switch (cfg) {
    case 0: return run<512, 32768, 6>(flags, x, y, n, ws, s, grid_out);
    case 1: return run<512, 32768, 4>(flags, x, y, n, ws, s, grid_out);
    case 2: return run<512, 16384, 12>(flags, x, y, n, ws, s, grid_out);
    case 3: return run<1024, 65536, 3>(flags, x, y, n, ws, s, grid_out);
    case 4: return run<256, 16384, 6>(flags, x, y, n, ws, s, grid_out);   // 2 CTAs / SM
    case 5: return run<512, 32768, 3>(flags, x, y, n, ws, s, grid_out);   // 2 CTAs / SM
    case 6: return run<256, 32768, 6>(flags, x, y, n, ws, s, grid_out);   // V = 8
    case 10: return run_ws<16, 32768, 6>(flags, x, y, n, ws, s, grid_out);
    case 11: return run_ws<16, 32768, 4>(flags, x, y, n, ws, s, grid_out);
    case 12: return run_ws<8, 32768, 6>(flags, x, y, n, ws, s, grid_out);
    case 13: return run_ws<16, 65536, 3>(flags, x, y, n, ws, s, grid_out);
    case 14: return run_ws<32, 65536, 3>(flags, x, y, n, ws, s, grid_out);
    case 15: return run_ws<8, 16384, 12>(flags, x, y, n, ws, s, grid_out);
    case 16: return run_ws<16, 16384, 12>(flags, x, y, n, ws, s, grid_out);
    case 17: return run_ws<16, 32768, 7>(flags, x, y, n, ws, s, grid_out);
    case 18: return run_ws<8, 32768, 7>(flags, x, y, n, ws, s, grid_out);
    case 19: return run_ws<16, 65536, 3>(flags, x, y, n, ws, s, grid_out);
    case 20: return run_ws<16, 32768, 5>(flags, x, y, n, ws, s, grid_out);
    case 30: return run_ws<16, 32768, 4, 2>(flags, x, y, n, ws, s, grid_out);
    case 31: return run_ws<16, 32768, 5, 2>(flags, x, y, n, ws, s, grid_out);
    case 32: return run_ws<16, 32768, 6, 2>(flags, x, y, n, ws, s, grid_out);
    case 33: return run_ws<16, 32768, 7, 2>(flags, x, y, n, ws, s, grid_out);
    case 34: return run_ws<8, 32768, 6, 2>(flags, x, y, n, ws, s, grid_out);
    case 35: return run_ws<16, 65536, 3, 2>(flags, x, y, n, ws, s, grid_out);
    case 36: return run_ws<16, 16384, 12, 2>(flags, x, y, n, ws, s, grid_out);
    case 37: return run_ws<8, 16384, 12, 2>(flags, x, y, n, ws, s, grid_out);
    case 38: return run_ws<24, 49152, 4, 2>(flags, x, y, n, ws, s, grid_out);
    case 39: return run_ws<16, 32768, 6, 1>(flags, x, y, n, ws, s, grid_out);
    case 40: return run_ws<12, 49152, 4, 2>(flags, x, y, n, ws, s, grid_out);
    case 41: return run_ws<8, 32768, 5, 2>(flags, x, y, n, ws, s, grid_out);
    case 42: return run_ws<8, 32768, 4, 2>(flags, x, y, n, ws, s, grid_out);
    }
    return -3;
}
