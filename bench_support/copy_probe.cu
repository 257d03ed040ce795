// copy_probe.cu — HBM ceiling probes for bench.py (NOT the product path).
//
// The scan moves exactly 2N·sizeof(T) bytes (read x once, write y once), so
// its roofline is the fastest device-to-device copy this GPU can run.  The
// driver's MEASURED_PEAKS.json figure is a torch copy_; the scan reached
// 1.00–1.04 of it in round 1, so the true ceiling was unknown.  Four probes,
// each timed by bench.py with CUDA events on the launching stream:
//
//   probe_tma_copy   the scan kernel's own data movement with no compute:
//                    persistent CTAs (one per SM), 1-D TMA bulk loads
//                    (cp.async.bulk) into a STAGES-deep shared-memory ring,
//                    1-D TMA bulk stores straight back out of the ring
//   probe_vec_copy   grid-stride 256-bit loads / stores through registers
//                    (the scan's scanner warps use the same STG.E.ENL2.256)
//   probe_memcpy     cudaMemcpyAsync device-to-device (the copy engines /
//                    the driver's own copy kernel)
//   probe_read       read-only: 256-bit loads folded into a checksum (the
//                    read half of the traffic on its own)
#include <cstdint>
#include <cuda_runtime.h>

#include "lscan_ptx.cuh"

using namespace lscan;

namespace {

template <int TILE, int STAGES>
__global__ void __launch_bounds__(32, 1) tma_copy_kernel(const uint8_t *x, uint8_t *y, int64_t tiles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * TILE);
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t mine = (tiles - c + G - 1) / G;
    if (threadIdx.x != 0) return;
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
    const uint64_t pol = policy_evict_first();
    auto load = [&](int64_t k) {
        const int s = (int)(k % STAGES);
        mbar_arrive_expect_tx(&full[s], TILE);
        tma_load_1d(smem + s * TILE, x + (c + k * G) * TILE, TILE, &full[s], pol);
    };
    for (int64_t k = 0; k < STAGES && k < mine; ++k) load(k);
    for (int64_t k = 0; k < mine; ++k) {
        const int s = (int)(k % STAGES);
        mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
        tma_store_1d(y + (c + k * G) * TILE, smem + s * TILE, TILE, pol);
        bulk_commit();
        // the previous tile's store has read its stage: refill that stage
        if (k >= 1 && k - 1 + STAGES < mine) {
            bulk_wait_read<1>();
            load(k - 1 + STAGES);
        }
    }
    bulk_wait_all();
}

__global__ void __launch_bounds__(256) vec_copy_kernel(const uint8_t *x, uint8_t *y, int64_t chunks) {
    // one 32-byte chunk per lane per iteration, 4 in flight
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 3 * stride < chunks; i += 4 * stride) {
        uint4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg256(x + (i + u * stride) * 32, a[u], b[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) stg256(y + (i + u * stride) * 32, a[u], b[u]);
    }
    for (; i < chunks; i += stride) {
        uint4 a, b;
        ldg256(x + i * 32, a, b);
        stg256(y + i * 32, a, b);
    }
}

__global__ void __launch_bounds__(256) read_kernel(const uint8_t *x, int64_t chunks, unsigned *sink) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned acc = 0;
    for (; i + 3 * stride < chunks; i += 4 * stride) {
        uint4 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) ldg256(x + (i + u * stride) * 32, a[u], b[u]);
#pragma unroll
        for (int u = 0; u < 4; ++u) acc ^= a[u].x ^ a[u].y ^ a[u].z ^ a[u].w ^ b[u].x ^ b[u].y ^ b[u].z ^ b[u].w;
    }
    for (; i < chunks; i += stride) {
        uint4 a, b;
        ldg256(x + i * 32, a, b);
        acc ^= a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w;
    }
    if (acc == 0x9e3779b9u) *sink = acc;  // practically never: keeps the loads alive
}

constexpr int kTile = 32768, kStages = 6;

int sms() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return n;
}

}  // namespace

extern "C" {

// bytes must be a multiple of 32 KiB for the TMA probe and of 32 for the
// others; x and y 1024-byte aligned (torch allocations are)
int probe_tma_copy(const void *x, void *y, int64_t bytes, void *stream) {
    auto fn = tma_copy_kernel<kTile, kStages>;
    const size_t smem = (size_t)kStages * kTile + kStages * 8;
    if (cudaFuncSetAttribute((const void *)fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
        return 1;
    const int64_t tiles = bytes / kTile;
    fn<<<sms(), 32, smem, static_cast<cudaStream_t>(stream)>>>(static_cast<const uint8_t *>(x),
                                                                static_cast<uint8_t *>(y), tiles);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int probe_vec_copy(const void *x, void *y, int64_t bytes, int blocks_per_sm, void *stream) {
    vec_copy_kernel<<<sms() * blocks_per_sm, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t *>(x), static_cast<uint8_t *>(y), bytes / 32);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

int probe_memcpy(const void *x, void *y, int64_t bytes, void *stream) {
    return cudaMemcpyAsync(y, x, (size_t)bytes, cudaMemcpyDeviceToDevice, static_cast<cudaStream_t>(stream)) ==
                   cudaSuccess
               ? 0
               : 2;
}

int probe_read(const void *x, int64_t bytes, void *sink, int blocks_per_sm, void *stream) {
    read_kernel<<<sms() * blocks_per_sm, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint8_t *>(x), bytes / 32, static_cast<unsigned *>(sink));
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}

}  // extern "C"
