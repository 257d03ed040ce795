// clock_probe.cu — laboratory (NOT the product): the SM clock each SM really
// runs at, from clock64() cycles over %globaltimer nanoseconds while a block
// spins for `spin_ns`.  Used to tell a clock (power / thermal) slowdown from
// a memory-side one when a kernel's throughput drifts under sustained load.
#include <cuda_runtime.h>

#include <cstdint>

__global__ void clock_probe_kernel(long long *out, long long spin_ns) {
    if (threadIdx.x != 0) return;
    uint64_t t0, t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    const long long c0 = clock64();
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    } while ((long long)(t1 - t0) < spin_ns);
    const long long c1 = clock64();
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    out[3 * blockIdx.x + 0] = smid;
    out[3 * blockIdx.x + 1] = c1 - c0;
    out[3 * blockIdx.x + 2] = (long long)(t1 - t0);
}

extern "C" int clock_probe(long long *out_dev, int blocks, long long spin_ns, void *stream) {
    clock_probe_kernel<<<blocks, 32, 0, static_cast<cudaStream_t>(stream)>>>(out_dev, spin_ns);
    return (int)cudaGetLastError();
}
