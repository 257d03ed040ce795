// cub_side.cu — side reference for bench.py only (NOT the product path):
// cub::DeviceScan::InclusiveSum (CUB 2.8.2, CUDA 12.9) on the same device
// buffers, so the bench can print CUB's Gelem/s next to ours.
#include <cstdint>
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

namespace {
template <typename T>
int run(const void *x, void *y, int64_t n, void *temp, size_t *temp_bytes, cudaStream_t s) {
    cudaError_t e = cub::DeviceScan::InclusiveSum(temp, *temp_bytes, static_cast<const T *>(x), static_cast<T *>(y),
                                                  n, s);
    return e == cudaSuccess ? 0 : (int)e;
}
}  // namespace

extern "C" {
// dt: 0 = i32, 1 = i64, 2 = f32, 3 = f64 (ls_dtype).  temp == NULL -> query.
int cub_inclusive_sum(int dt, const void *x, void *y, int64_t n, void *temp, size_t *temp_bytes, void *stream) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dt) {
    case 0: return run<int32_t>(x, y, n, temp, temp_bytes, s);
    case 1: return run<int64_t>(x, y, n, temp, temp_bytes, s);
    case 2: return run<float>(x, y, n, temp, temp_bytes, s);
    case 3: return run<double>(x, y, n, temp, temp_bytes, s);
    }
    return -1;
}
}
