// lscan_host.cu — ls_inclusive_sum_host: the numpy-facing drop-in path.
//
// The reference's chained_scan(problem) takes host (numpy) arrays and
// returns host arrays (chainscan/chained.py:316-357, reference.py:38-58).
// This entry keeps that contract on a GPU: the array is cut into chunks that
// are streamed host->device, scanned in place on the device with the carry
// chained through two device scalars, and streamed device->host, with the
// three stages of consecutive chunks overlapped on three CUDA streams
// (copy-in / scan / copy-out), so the wall time approaches the slower PCIe
// direction rather than the sum of the three.
//
// Pinned host buffers (cudaHostAlloc / cudaHostRegister / torch pin_memory)
// are DMA'd directly.  Pageable buffers go through per-chunk pinned staging
// buffers; the calling thread does the host memcpy for chunk k while the
// device works on the DMA and scan of chunk k-1.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "lscan.h"

namespace lscan {
void set_detail(const std::string &msg);
}

namespace {

constexpr int kBufs = 3;
constexpr size_t kDefaultChunkMiB = 32;  // per-chunk bytes; LSCAN_HOST_CHUNK_MB overrides

size_t chunk_bytes_from_env() {
    const char *e = getenv("LSCAN_HOST_CHUNK_MB");
    long mb = e ? atol(e) : (long)kDefaultChunkMiB;
    if (mb < 1) mb = 1;
    if (mb > 1024) mb = 1024;
    return (size_t)mb << 20;
}

struct HostCtx {
    bool init = false;
    int device = -1;
    cudaStream_t s_in = nullptr, s_comp = nullptr, s_out = nullptr;
    void *dbuf[kBufs] = {};
    void *pin_in[kBufs] = {};
    void *pin_out[kBufs] = {};
    void *carry = nullptr;  // two scalar slots (ping-pong), 16 B each
    void *ws = nullptr;
    size_t ws_bytes = 0;
    cudaEvent_t ev_in[kBufs] = {}, ev_comp[kBufs] = {}, ev_out[kBufs] = {};
    size_t chunk_bytes = 0;
    std::mutex mu;
};

std::mutex g_ctx_mu;
std::vector<HostCtx *> g_ctx;

ls_status host_fail(ls_status s, cudaError_t e, const char *what) {
    lscan::set_detail(std::string(what) + ": " + cudaGetErrorString(e));
    return s;
}

#define HC(call, what)                                            \
    do {                                                          \
        cudaError_t e_ = (call);                                  \
        if (e_ != cudaSuccess) return host_fail(LS_ERR_CUDA, e_, what); \
    } while (0)

ls_status ctx_for(int dev, HostCtx **out) {
    std::lock_guard<std::mutex> lk(g_ctx_mu);
    if ((int)g_ctx.size() <= dev) g_ctx.resize(dev + 1, nullptr);
    if (!g_ctx[dev]) g_ctx[dev] = new HostCtx();
    HostCtx *c = g_ctx[dev];
    if (!c->init) {
        c->device = dev;
        c->chunk_bytes = chunk_bytes_from_env();
        const size_t kChunkBytes = c->chunk_bytes;
        HC(cudaStreamCreateWithFlags(&c->s_in, cudaStreamNonBlocking), "stream");
        HC(cudaStreamCreateWithFlags(&c->s_comp, cudaStreamNonBlocking), "stream");
        HC(cudaStreamCreateWithFlags(&c->s_out, cudaStreamNonBlocking), "stream");
        for (int b = 0; b < kBufs; ++b) {
            HC(cudaMalloc(&c->dbuf[b], kChunkBytes), "chunk buffer");
            HC(cudaEventCreateWithFlags(&c->ev_in[b], cudaEventDisableTiming), "event");
            HC(cudaEventCreateWithFlags(&c->ev_comp[b], cudaEventDisableTiming), "event");
            HC(cudaEventCreateWithFlags(&c->ev_out[b], cudaEventDisableTiming), "event");
        }
        HC(cudaMalloc(&c->carry, 32), "carry scalars");
        c->ws_bytes = std::max(ls_workspace_bytes(LS_I32, (int64_t)(kChunkBytes / 4)),
                               ls_workspace_bytes(LS_I64, (int64_t)(kChunkBytes / 8)));
        HC(cudaMalloc(&c->ws, c->ws_bytes), "workspace");
        if (ls_workspace_init(c->ws, c->ws_bytes, c->s_comp) != LS_OK) return LS_ERR_CUDA;
        HC(cudaStreamSynchronize(c->s_comp), "workspace init");
        c->init = true;
    }
    *out = c;
    return LS_OK;
}

ls_status ensure_staging(HostCtx *c) {
    const size_t kChunkBytes = c->chunk_bytes;
    for (int b = 0; b < kBufs; ++b) {
        if (!c->pin_in[b]) HC(cudaHostAlloc(&c->pin_in[b], kChunkBytes, cudaHostAllocDefault), "pinned staging");
        if (!c->pin_out[b]) HC(cudaHostAlloc(&c->pin_out[b], kChunkBytes, cudaHostAllocDefault), "pinned staging");
    }
    return LS_OK;
}

bool is_pinned(const void *p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

int esize(ls_dtype dt) { return (dt == LS_I32 || dt == LS_F32) ? 4 : 8; }

// Host copy between pageable memory and the pinned staging buffers, split
// over a few threads: a single core's memcpy (~5-10 GB/s) would otherwise
// bound the pageable pipeline well below PCIe.
void parallel_memcpy(void *dst, const void *src, size_t bytes) {
    static const unsigned hw = std::thread::hardware_concurrency();
    static const unsigned cap = [] {
        const char *e = getenv("LSCAN_HOST_COPY_THREADS");
        return e ? (unsigned)std::max(1, atoi(e)) : 16u;  // 16 measured 5 % faster than 8 (scripts/gpu_pageable_threads.sh)
    }();
    const unsigned nt = std::max(1u, std::min(cap, hw ? hw : 1u));
    if (bytes < ((size_t)4 << 20) || nt == 1) {
        memcpy(dst, src, bytes);
        return;
    }
    // ceil(bytes / nt) rounded up to a page: nt parts always cover every byte
    // (floor(bytes / nt) already page-aligned would leave bytes % nt uncopied)
    const size_t part = (((bytes + nt - 1) / nt) + 4095) & ~(size_t)4095;
    std::vector<std::thread> th;
    for (unsigned i = 1; i < nt; ++i) {
        const size_t off = part * i;
        if (off >= bytes) break;
        const size_t len = std::min(part, bytes - off);
        th.emplace_back([=] { memcpy((char *)dst + off, (const char *)src + off, len); });
    }
    memcpy(dst, src, std::min(part, bytes));
    for (auto &t : th) t.join();
}

// The chunk pipeline proper.  Returns at the first failure; the caller
// (ls_scan_host_ex) synchronises the three streams and restores the device
// on every path, so no copy is still writing into y or the staging buffers
// when an error is reported.
ls_status run_pipeline(HostCtx *c, ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, int flags) {
    const int es = esize(dt);
    const bool exclusive = (flags & LS_HOST_EXCLUSIVE) != 0;
    const bool ordered = (flags & LS_HOST_ORDERED) != 0;
    ls_status st = LS_OK;
    const bool direct = is_pinned(x) && is_pinned(y);
    if (!direct && (st = ensure_staging(c)) != LS_OK) return st;

    const int64_t chunk = (int64_t)(c->chunk_bytes / es);
    const int64_t nchunks = (n + chunk - 1) / chunk;
    const uint8_t *xb = static_cast<const uint8_t *>(x);
    uint8_t *yb = static_cast<uint8_t *>(y);
    uint8_t *carry = static_cast<uint8_t *>(c->carry);

    auto drain = [&](int64_t k) -> ls_status {
        // finish chunk k on the host side (pageable path only)
        const int b = (int)(k % kBufs);
        const int64_t off = k * chunk, len = std::min(chunk, n - off);
        HC(cudaEventSynchronize(c->ev_out[b]), "copy-out wait");
        parallel_memcpy(yb + off * es, c->pin_out[b], (size_t)len * es);
        return LS_OK;
    };

    for (int64_t k = 0; k < nchunks; ++k) {
        const int b = (int)(k % kBufs);
        const int64_t off = k * chunk, len = std::min(chunk, n - off);
        const size_t bytes = (size_t)len * es;
        if (k >= kBufs) {
            // buffer b is free once chunk k - kBufs has left the device
            if (!direct && (st = drain(k - kBufs)) != LS_OK) return st;
            HC(cudaStreamWaitEvent(c->s_in, c->ev_out[b], 0), "wait buffer");
        }
        const void *src = xb + off * es;
        if (!direct) {
            if (k >= kBufs) HC(cudaEventSynchronize(c->ev_in[b]), "staging reuse");
            parallel_memcpy(c->pin_in[b], src, bytes);
            src = c->pin_in[b];
        }
        HC(cudaMemcpyAsync(c->dbuf[b], src, bytes, cudaMemcpyHostToDevice, c->s_in), "copy-in");
        HC(cudaEventRecord(c->ev_in[b], c->s_in), "event");
        HC(cudaStreamWaitEvent(c->s_comp, c->ev_in[b], 0), "wait copy-in");
        const void *cin = k ? carry + 16 * ((k - 1) & 1) : nullptr;
        void *cout = carry + 16 * (k & 1);
        if (ordered)
            st = ls_ordered_scan(op, dt, c->dbuf[b], c->dbuf[b], len, exclusive ? 1 : 0, cin, cout, c->s_comp);
        else if (exclusive)
            st = ls_exclusive_scan(op, dt, c->dbuf[b], c->dbuf[b], len, cin, cout, c->ws, c->ws_bytes, c->s_comp);
        else
            st = ls_inclusive_scan(op, dt, c->dbuf[b], c->dbuf[b], len, cin, cout, c->ws, c->ws_bytes, c->s_comp);
        if (st != LS_OK) return st;
        HC(cudaEventRecord(c->ev_comp[b], c->s_comp), "event");
        HC(cudaStreamWaitEvent(c->s_out, c->ev_comp[b], 0), "wait scan");
        void *dst = direct ? (void *)(yb + off * es) : c->pin_out[b];
        HC(cudaMemcpyAsync(dst, c->dbuf[b], bytes, cudaMemcpyDeviceToHost, c->s_out), "copy-out");
        HC(cudaEventRecord(c->ev_out[b], c->s_out), "event");
    }
    if (!direct) {
        for (int64_t k = std::max<int64_t>(0, nchunks - kBufs); k < nchunks; ++k)
            if ((st = drain(k)) != LS_OK) return st;
    }
    return LS_OK;
}

}  // namespace

extern "C" ls_status ls_scan_host_ex(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, int flags,
                                     int device) {
    if (dt < LS_I32 || dt > LS_F64 || op < LS_OP_ADD || op > LS_OP_MIN) return LS_ERR_UNSUPPORTED_DTYPE;
    if (n < 0 || (n > 0 && (!x || !y)) || (flags & ~(LS_HOST_EXCLUSIVE | LS_HOST_ORDERED))) return LS_ERR_INVALID_ARG;
    if (n == 0) return LS_OK;
    const int es = esize(dt);
    if (x != y) {
        const uintptr_t a = (uintptr_t)x, b = (uintptr_t)y, bytes = (uintptr_t)n * es;
        if (a < b + bytes && b < a + bytes) return LS_ERR_INVALID_ARG;
    }
    int prev = 0;
    HC(cudaGetDevice(&prev), "cudaGetDevice");
    int dev = device < 0 ? prev : device;
    if (prev != dev) HC(cudaSetDevice(dev), "cudaSetDevice");
    HostCtx *c = nullptr;
    ls_status st = ctx_for(dev, &c);
    if (st == LS_OK) {
        std::lock_guard<std::mutex> lk(c->mu);
        st = run_pipeline(c, op, dt, x, y, n, flags);
        // one exit for every outcome: nothing of this call is still in flight
        // when it returns, error or not
        const cudaError_t e_out = cudaStreamSynchronize(c->s_out);
        const cudaError_t e_comp = cudaStreamSynchronize(c->s_comp);
        const cudaError_t e_in = cudaStreamSynchronize(c->s_in);
        if (st == LS_OK) {
            if (e_out != cudaSuccess) st = host_fail(LS_ERR_CUDA, e_out, "final sync (copy-out)");
            else if (e_comp != cudaSuccess) st = host_fail(LS_ERR_CUDA, e_comp, "final sync (scan)");
            else if (e_in != cudaSuccess) st = host_fail(LS_ERR_CUDA, e_in, "final sync (copy-in)");
        }
    }
    if (prev != dev) {
        const cudaError_t e = cudaSetDevice(prev);
        if (st == LS_OK && e != cudaSuccess) st = host_fail(LS_ERR_CUDA, e, "cudaSetDevice (restore)");
    }
    return st;
}

extern "C" ls_status ls_scan_host(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, int exclusive,
                                  int device) {
    return ls_scan_host_ex(op, dt, x, y, n, exclusive ? LS_HOST_EXCLUSIVE : 0, device);
}

extern "C" ls_status ls_inclusive_sum_host(ls_dtype dt, const void *x, void *y, int64_t n, int exclusive,
                                           int device) {
    return ls_scan_host(LS_OP_ADD, dt, x, y, n, exclusive, device);
}
