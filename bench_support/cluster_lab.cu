// cluster_lab.cu — laboratory for the small-n latency kernel (NOT the
// product): geometry variants of lscan::scan_cluster_kernel and a plain
// load/store kernel of the same shape (the floor for "read 4 vectors per
// thread, write them back"), launched with one cluster per call.
//
//   lab_cluster(variant, x, y, n, ws, coop, stream) -> 0 / CUDA error code
//     0: 256 threads, 4 rows (product)    1: 512 threads, 4 rows
//     2: 256 threads, 8 rows              3: 256 threads, 2 rows
//     4: copy 1024 x 4 rows               5: copy 256 x 4 rows
//     6: 256 x 16 rows (2 blocks/SM)       7: 256 x 8 rows (2 blocks/SM, product mid)
//     8: int64 256 x 4 (product small)     9: int64 256 x 8 (product mid)
//    10: int64 512 x 4 (2 blocks/SM)       11: int64 512 x 2
//    12: 256 x 16 rows (1 block/SM)        13: int64 256 x 16 (1 block/SM)
//    14: int64 256 x 12 (product large)    15: 256 x 12 (product large)
//    16..21: 32-byte lane rows (VW = 2): 256x4, 256x8 minb2, i64 256x4, i64 256x8 minb2,
//            i64 256x12 minb2, 256x12 minb2
//    22..24: i64, 512 threads, VW = 2: 4 rows minb2, 8 rows minb1, 6 rows minb1
//    25, 26: f64 256 x 8 minb2, 256 x 12 minb2 (the product mid / large geometries)
//   lab_block_elems(variant) -> elements per block (int32)
#include <cuda_runtime.h>

#include "lscan_cluster.cuh"

using namespace lscan;

template <int THREADS, int V>
__global__ void __launch_bounds__(THREADS, 1) copy_kernel(const ScanParams p) {
    constexpr int WARP_VECS = 32 * V;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t t0 = (int64_t)blockIdx.x * (THREADS / 32) * WARP_VECS * 4;
    const int64_t valid = p.n - t0;
    const int32_t *x = static_cast<const int32_t *>(p.x) + t0;
    int32_t *y = static_cast<int32_t *>(p.y) + t0;
    uint4 d[V];
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int64_t e0 = (int64_t)(warp * WARP_VECS + j * 32 + lane) * 4;
        d[j] = e0 + 4 <= valid ? ldg128(x + e0) : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int j = 0; j < V; ++j) {
        const int64_t e0 = (int64_t)(warp * WARP_VECS + j * 32 + lane) * 4;
        if (e0 + 4 <= valid) stg128_v4(y + e0, d[j]);
    }
}

namespace {
struct Var {
    void (*fn)(const ScanParams);
    int threads;
    int rows;
    int es = 4;  // element size
};
Var var(int v) {
    switch (v) {
    case 0: return {&scan_cluster_kernel<int32_t, OpAdd, false, 4, 256, 4>, 256, 4};
    case 1: return {&scan_cluster_kernel<int32_t, OpAdd, false, 4, 512, 2>, 512, 4};
    case 2: return {&scan_cluster_kernel<int32_t, OpAdd, false, 8, 256, 4>, 256, 8};
    case 3: return {&scan_cluster_kernel<int32_t, OpAdd, false, 2, 256, 4>, 256, 2};
    case 4: return {&copy_kernel<1024, 4>, 1024, 4};
    case 5: return {&copy_kernel<256, 4>, 256, 4};
    case 6: return {&scan_cluster_kernel<int32_t, OpAdd, false, 16, 256, 2>, 256, 16};
    case 7: return {&scan_cluster_kernel<int32_t, OpAdd, false, 8, 256, 2>, 256, 8};
    // 64-bit elements, small and mid geometry
    case 8: return {&scan_cluster_kernel<int64_t, OpAdd, false, 4, 256, 4>, 256, 4, 8};
    case 9: return {&scan_cluster_kernel<int64_t, OpAdd, false, 8, 256, 2>, 256, 8, 8};
    case 10: return {&scan_cluster_kernel<int64_t, OpAdd, false, 4, 512, 2>, 512, 4, 8};
    case 11: return {&scan_cluster_kernel<int64_t, OpAdd, false, 2, 512, 4>, 512, 2, 8};
    case 12: return {&scan_cluster_kernel<int32_t, OpAdd, false, 16, 256, 1>, 256, 16};
    case 13: return {&scan_cluster_kernel<int64_t, OpAdd, false, 16, 256, 1>, 256, 16, 8};
    case 14: return {&scan_cluster_kernel<int64_t, OpAdd, false, 12, 256, 2>, 256, 12, 8};
    case 15: return {&scan_cluster_kernel<int32_t, OpAdd, false, 12, 256, 2>, 256, 12};
    case 16: return {&scan_cluster_kernel<int32_t, OpAdd, false, 4, 256, 4, 2>, 256, 4};
    case 17: return {&scan_cluster_kernel<int32_t, OpAdd, false, 8, 256, 2, 2>, 256, 8};
    case 18: return {&scan_cluster_kernel<int64_t, OpAdd, false, 4, 256, 4, 2>, 256, 4, 8};
    case 19: return {&scan_cluster_kernel<int64_t, OpAdd, false, 8, 256, 2, 2>, 256, 8, 8};
    case 20: return {&scan_cluster_kernel<int64_t, OpAdd, false, 12, 256, 2, 2>, 256, 12, 8};
    case 21: return {&scan_cluster_kernel<int32_t, OpAdd, false, 12, 256, 2, 2>, 256, 12};
    case 22: return {&scan_cluster_kernel<int64_t, OpAdd, false, 4, 512, 2, 2>, 512, 4, 8};
    case 23: return {&scan_cluster_kernel<int64_t, OpAdd, false, 8, 512, 1, 2>, 512, 8, 8};
    case 24: return {&scan_cluster_kernel<int64_t, OpAdd, false, 6, 512, 1, 2>, 512, 6, 8};
    // f64 on the product mid / large geometries (as 19 / 20 for i64)
    case 25: return {&scan_cluster_kernel<double, OpAdd, false, 8, 256, 2, 2>, 256, 8, 8};
    default: return {&scan_cluster_kernel<double, OpAdd, false, 12, 256, 2, 2>, 256, 12, 8};
    }
}
}  // namespace

namespace {
void *g_ctl = nullptr;  // LS_LAB_CTIMELINE builds: per-block event times
int g_csize = 16;       // blocks per cluster
}  // namespace

extern "C" {
void lab_set_timeline(void *buf) { g_ctl = buf; }
void lab_set_cluster_size(int c) { g_csize = c; }
long long lab_block_elems(int v) {
    const Var w = var(v);
    return (long long)w.threads * w.rows * 16 / w.es;
}

// ws: a zeroed workspace (needed when n spans several clusters); coop: 0
// drops the cooperative attribute (measures its cost; unsafe in general)
int lab_cluster(int v, const void *x, void *y, long long n, void *ws, int coop, void *stream) {
    const Var w = var(v);
    const long long be = lab_block_elems(v);
    const long long tiles = (n + be - 1) / be;
    const int C = (int)(tiles < g_csize ? tiles : g_csize);
    const long long K = (tiles + C - 1) / C;
    if (C < 1 || (K > 1 && ((v == 4 || v == 5) || !ws))) return -1;
    static bool init[32] = {};  // variants 0..26
    if (!init[v]) {
        cudaFuncSetAttribute((const void *)w.fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        init[v] = true;
    }
    ScanParams p{};
    p.x = x;
    p.y = y;
    p.n = n;
    p.ws = static_cast<uint8_t *>(ws);
    p.xchg = static_cast<uint8_t *>(g_ctl);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(K * C));
    cfg.blockDim = dim3((unsigned)w.threads);
    cfg.stream = static_cast<cudaStream_t>(stream);
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeCooperative;
    attr[1].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = (K > 1 && coop) ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, w.fn, p);
    if (e != cudaSuccess) (void)cudaGetLastError();  // e.g. a grid too large to be co-resident
    return (int)e;
}
}
