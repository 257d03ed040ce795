// lscan_ordered.cuh — the strict left fold on the device: the reference's
// B = 1 path (chainscan/chained.py:290-313, "carry prepended, then one fused
// accumulate"), which defines float bit-exactness against the sequential
// oracle (reference.py:61-67; test_chained.py:221-226, test_acceptance.py:85-111).
//
// Float addition is not associative, so the B = 1 result — every y[j]
// rounded from y[j-1] + x[j] — has no parallel formulation that reproduces
// its bits.  This kernel runs that chain on the device at the speed of the
// dependent add (one FADD / DADD latency per element), with the memory
// traffic fully off the chain:
//
//   producer warp  1-D TMA bulk loads (cp.async.bulk) of x into a ring of
//                  16 KiB stages, completion on mbarriers
//   folder         one thread: acc = acc (+) x[j] for every element of a
//                  landed stage, results written back in place (the chain)
//   storer warps   coalesced stores of a folded stage to y (any alignment)
//
// Elements before x's first 16-byte boundary and after its last one are
// folded straight from global memory by the folder.  x == y is safe: the
// folder reads x[j] before anything writes y[j], and the producer never
// loads a stage the storers have written.  One CTA; the launch is on the
// caller's stream like every other scan.
#pragma once
#include "lscan_common.cuh"

namespace lscan {

__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }

constexpr int kOrdStageBytes = 16384, kOrdStages = 8, kOrdThreads = 128;
constexpr size_t kOrdSmemBytes = (size_t)kOrdStages * kOrdStageBytes + 3 * kOrdStages * 8;

template <typename T, typename OP, bool EXCL>
__global__ void __launch_bounds__(kOrdThreads, 1) scan_ordered_kernel(const ScanParams p) {
    constexpr int PER = 16 / (int)sizeof(T);
    constexpr int STORERS = kOrdThreads - 64;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + kOrdStages * kOrdStageBytes);
    uint64_t *folded = full + kOrdStages;
    uint64_t *empty = folded + kOrdStages;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const T *x = static_cast<const T *>(p.x);
    T *y = static_cast<T *>(p.y);
    const int64_t n = p.n;
    const T ident = OP::template identity<T>();

    // the first element is folded on its own (it seeds the chain: y[0] = x[0]
    // exactly without a carry, as numpy's accumulate copies it); the rest
    // splits into head (to x's 16-byte boundary), body (whole vectors through
    // the ring) and tail
    const int64_t first = 1;
    const uintptr_t xa = (uintptr_t)(x + first);
    const int64_t head = n <= first ? 0 : imin64(n - first, (int64_t)(((16 - (xa & 15u)) & 15u) / sizeof(T)));
    const int64_t b0 = first + head;  // first body element
    const int64_t body = n > b0 ? ((n - b0) / PER) * PER : 0;
    const int64_t nstages = (body * (int64_t)sizeof(T) + kOrdStageBytes - 1) / kOrdStageBytes;

    if (tid == 0) {
        for (int s = 0; s < kOrdStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&folded[s], 1);
            mbar_init(&empty[s], STORERS);
        }
        fence_mbar_init();
    }
    __syncthreads();
    if (n <= 0) return;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            const uint64_t pol = policy_evict_first();
            const uint8_t *xb = reinterpret_cast<const uint8_t *>(x + b0);
            const int64_t bbytes = body * (int64_t)sizeof(T);
            for (int64_t k = 0; k < nstages; ++k) {
                const int s = (int)(k % kOrdStages);
                if (k >= kOrdStages) mbar_wait(&empty[s], (uint32_t)(((k / kOrdStages) - 1) & 1));
                const int64_t off = k * kOrdStageBytes;
                const uint32_t bytes = (uint32_t)imin64(kOrdStageBytes, bbytes - off);
                mbar_arrive_expect_tx(&full[s], bytes);
                tma_load_1d(smem + s * kOrdStageBytes, xb + off, bytes, &full[s], pol);
            }
        }
    } else if (warp == 1) {
        // -------------------------------------------------------------- folder
        if (lane == 0) {
            const T *cin = static_cast<const T *>(p.carry_in);
            T acc;
            {
                const T v = x[0];
                if (cin != nullptr) {
                    const T c = *cin;
                    y[0] = EXCL ? c : OP::apply(c, v);
                    acc = OP::apply(c, v);
                } else {
                    y[0] = EXCL ? ident : v;
                    acc = v;
                }
            }
            for (int64_t j = first; j < b0; ++j) {
                const T v = x[j];
                if (EXCL) y[j] = acc;
                acc = OP::apply(acc, v);
                if (!EXCL) y[j] = acc;
            }
            const int64_t bbytes = body * (int64_t)sizeof(T);
            for (int64_t k = 0; k < nstages; ++k) {
                const int s = (int)(k % kOrdStages);
                mbar_wait(&full[s], (uint32_t)((k / kOrdStages) & 1));
                const int nvec = (int)(imin64(kOrdStageBytes, bbytes - k * kOrdStageBytes) / 16);
                uint4 *st = reinterpret_cast<uint4 *>(smem + s * kOrdStageBytes);
                int v = 0;
                // plain shared accesses (no asm volatile): the compiler hoists
                // the loads of a group ahead of its dependent chain
                for (; v + 4 <= nvec; v += 4) {
                    Regs<T, 4> r;
#pragma unroll
                    for (int u = 0; u < 4; ++u) r.q[u] = st[v + u];
#pragma unroll
                    for (int e = 0; e < 4 * PER; ++e) {
                        const T xv = r.e[e];
                        if (EXCL) r.e[e] = acc;
                        acc = OP::apply(acc, xv);
                        if (!EXCL) r.e[e] = acc;
                    }
#pragma unroll
                    for (int u = 0; u < 4; ++u) st[v + u] = r.q[u];
                }
                for (; v < nvec; ++v) {
                    Regs<T, 1> r;
                    r.q[0] = st[v];
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        const T xv = r.e[e];
                        if (EXCL) r.e[e] = acc;
                        acc = OP::apply(acc, xv);
                        if (!EXCL) r.e[e] = acc;
                    }
                    st[v] = r.q[0];
                }
                // the stage is rewritten by TMA (async proxy) after the storers
                fence_proxy_async_smem();
                mbar_arrive(&folded[s]);
            }
            for (int64_t j = b0 + body; j < n; ++j) {
                const T v = x[j];
                if (EXCL) y[j] = acc;
                acc = OP::apply(acc, v);
                if (!EXCL) y[j] = acc;
            }
            if (p.total_out != nullptr) *static_cast<T *>(p.total_out) = acc;
        }
    } else {
        // -------------------------------------------------------------- storers
        const int st_id = tid - 64;
        const int64_t bbytes = body * (int64_t)sizeof(T);
        for (int64_t k = 0; k < nstages; ++k) {
            const int s = (int)(k % kOrdStages);
            mbar_wait(&folded[s], (uint32_t)((k / kOrdStages) & 1));
            const int cnt = (int)(imin64(kOrdStageBytes, bbytes - k * kOrdStageBytes) / (int64_t)sizeof(T));
            const T *src = reinterpret_cast<const T *>(smem + s * kOrdStageBytes);
            T *dst = y + b0 + k * (kOrdStageBytes / (int64_t)sizeof(T));
            for (int i = st_id; i < cnt; i += STORERS) dst[i] = src[i];
            mbar_arrive(&empty[s]);
        }
    }
}

}  // namespace lscan
