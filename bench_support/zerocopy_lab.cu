// zerocopy_lab.cu — laboratory (NOT the product): can kernels that read and
// write pinned host memory directly over PCIe (zero-copy, UVA) beat the
// DMA-engine pipeline of ls_scan_host (copy-in / scan / copy-out streams)?
//
//   zc_run(mode, hin, hout, dev, bytes, grid, threads, stream) -> cudaError_t
//     mode 0: read hin (host) -> dev          (PCIe read by SM loads)
//     mode 1: dev -> hout (host)              (PCIe write by SM stores)
//     mode 2: hin (host) -> hout (host)       (both directions in one kernel,
//                                              the access pattern of a
//                                              zero-copy scan)
//   zc_devptr(host) -> device alias of a pinned host pointer (or NULL)
#include <cuda_runtime.h>

#include <cstdint>

namespace {
__device__ __forceinline__ uint4 ld_v4(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

template <int U>
__global__ void zc_copy(const uint4 *__restrict__ src, uint4 *__restrict__ dst, size_t n16) {
    const size_t stride = (size_t)gridDim.x * blockDim.x * U;
    for (size_t base = ((size_t)blockIdx.x * blockDim.x) * U + threadIdx.x; base < n16; base += stride) {
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + (size_t)u * blockDim.x;
            if (i < n16) v[u] = ld_v4(src + i);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + (size_t)u * blockDim.x;
            if (i < n16) dst[i] = v[u];
        }
    }
}
}  // namespace

extern "C" {
void *zc_devptr(void *host) {
    void *d = nullptr;
    if (cudaHostGetDevicePointer(&d, host, 0) != cudaSuccess) {
        (void)cudaGetLastError();
        return nullptr;
    }
    return d;
}

int zc_run(int mode, void *hin, void *hout, void *dev, size_t bytes, int grid, int threads, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const size_t n16 = bytes / 16;
    const uint4 *src = static_cast<const uint4 *>(mode == 1 ? dev : hin);
    uint4 *dst = static_cast<uint4 *>(mode == 0 ? dev : hout);
    zc_copy<8><<<grid, threads, 0, s>>>(src, dst, n16);
    return (int)cudaGetLastError();
}
}
