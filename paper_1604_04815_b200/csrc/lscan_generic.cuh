// lscan_generic.cuh — the sequential persistent scan for arbitrary element
// alignment (pointers that are not 16-byte aligned cannot use TMA or 128-bit
// global accesses).
//
// One CTA runs the reference worker's per-block sequence in order
// (chainscan/chained.py:237-249): coalesced element loads of the tile into
// shared memory (identity-padded, partial_tail chained.py:188-202), a
// conflict-free register tile (rotated 128-bit shared loads), thread-serial +
// warp-shuffle + shared-memory block scan (Alg. 2/3), publish A[t], round
// look-back (the same slot protocol as the hot kernel), carry-seeded fold
// (Alg. 5), coalesced element stores.  The look-back sits on the critical
// path here, which is why the aligned hot path is warp-specialised
// (lscan_scan_ws2.cuh).
#pragma once
#include "lscan_common.cuh"

namespace lscan {

// Round look-back executed by one warp: prefix of tile t = r*G + c is
// R[r-1] (+) A[rG] (+) ... (+) A[rG+c-1], summed in a fixed order.
template <typename T, typename OP>
__device__ __forceinline__ bool round_lookback(const uint64_t *agg, const uint64_t *rnd, int64_t r, int c, int G,
                                               uint32_t tag, const T *carry_in, int lane, int64_t spin_budget,
                                               Header *hdr, T &prefix) {
    using S = Slot<T>;
    constexpr int U = 4;  // slots in flight per lane per pass
    T acc = OP::template identity<T>();
    int64_t probes = 0;
    bool dead = false;
    const int64_t base_t = r * (int64_t)G;
    for (int base = 0; base < c && !dead; base += 32 * U) {
        uint64_t w[U][S::W];
        bool need[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * 32 + lane;
            need[u] = j < c;
            if (need[u]) S::load(agg, base_t + j, w[u]);
        }
        T val[U];
        while (true) {
            bool ok = true;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (need[u]) {
                    if (S::decode(w[u], tag, val[u])) need[u] = false;
                    else ok = false;
                }
            }
            if (__all_sync(0xffffffffu, ok)) break;
            if (spin_budget > 0 && ++probes > spin_budget) {
                if (lane == 0) raise_error(hdr, 4u /*LS_ERR_LIVENESS*/, (uint32_t)(base_t + c));
                dead = true;
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (need[u]) { val[u] = OP::template identity<T>(); need[u] = false; }
                break;
            }
            __nanosleep(64);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = base + u * 32 + lane;
                if (need[u]) S::load(agg, base_t + j, w[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * 32 + lane;
            if constexpr (order_sensitive<T, OP>())
                acc = fold_chunk<T, OP>(acc, j < c ? val[u] : OP::template identity<T>());  // slot order
            else if (j < c)
                acc = OP::apply(acc, val[u]);  // lane-serial, ascending j
        }
    }
    const T asum = fold_finish<T, OP>(acc);
    bool has = false;
    T rp = OP::template identity<T>();
    if (r > 0) {
        uint64_t w[S::W];
        S::load(rnd, r - 1, w);
        while (!S::decode(w, tag, rp)) {
            if (spin_budget > 0 && ++probes > spin_budget) {
                if (lane == 0) raise_error(hdr, 4u, (uint32_t)(base_t + c));
                rp = OP::template identity<T>();
                break;
            }
            __nanosleep(64);
            S::load(rnd, r - 1, w);
        }
        has = true;
    } else if (carry_in != nullptr) {
        rp = *carry_in;
        has = true;
    }
    if (c > 0) {
        prefix = has ? OP::apply(rp, asum) : asum;
        return true;
    }
    prefix = rp;
    return has;
}

template <typename T, typename OP, int THREADS, int TILE_BYTES, bool EXCL>
__global__ void __launch_bounds__(THREADS, 1) scan_generic_kernel(const ScanParams p) {
    constexpr int NWARPS = THREADS / 32;
    constexpr int V = TILE_BYTES / THREADS / 16;    // 16-byte vectors per thread
    constexpr int ITEMS = V * 16 / (int)sizeof(T);  // elements per thread
    constexpr int TILE_ELEMS = TILE_BYTES / (int)sizeof(T);
    static_assert(V >= 1 && (V & (V - 1)) == 0, "vectors per thread must be a power of two");
    static_assert(NWARPS <= 32 && NWARPS >= 2, "2..32 warps");
    using S = Slot<T>;
    const T ident = OP::template identity<T>();

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *st = smem;
    T *warp_tot = reinterpret_cast<T *>(smem + TILE_BYTES);  // [NWARPS]
    T *warp_exc = warp_tot + NWARPS;                        // [NWARPS]
    T *tile_pre = warp_exc + NWARPS;                        // [1]
    int *tile_has = reinterpret_cast<int *>(tile_pre + 1);  // [1]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t M = p.num_tiles;
    Header *hdr = reinterpret_cast<Header *>(p.ws);
    uint64_t *agg = reinterpret_cast<uint64_t *>(p.ws + kSlotBase);
    uint64_t *rnd = agg + M * S::W;
    const T *x = static_cast<const T *>(p.x);
    T *y = static_cast<T *>(p.y);
    const T *carry_in = static_cast<const T *>(p.carry_in);
    const uint32_t tag = call_tag(hdr);
    const int64_t my_tiles = (M - c + G - 1) / G;

    for (int64_t k = 0; k < my_tiles; ++k) {
        const int64_t t = c + k * G;
        const int64_t t0 = t * TILE_ELEMS;
        int64_t valid = p.n - t0;
        if (valid > TILE_ELEMS) valid = TILE_ELEMS;
        T *sv = reinterpret_cast<T *>(st);
        for (int i = tid; i < TILE_ELEMS; i += THREADS) sv[i] = (i < valid) ? x[t0 + i] : ident;
        __syncthreads();

        Regs<T, V> r;
        load_tile_regs<T, V>(st, tid, r);
        T tsum = r.e[0];
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) tsum = OP::apply(tsum, r.e[i]);
        const T winc = warp_inclusive_scan<T, OP>(tsum, lane);
        const T wexc = __shfl_up_sync(0xffffffffu, winc, 1);
        if (lane == 31) warp_tot[warp] = winc;
        __syncthreads();  // (A)

        if (warp == 0) {
            const T wt = lane < NWARPS ? warp_tot[lane] : ident;
            const T wi = warp_inclusive_scan<T, OP>(wt, lane);
            const T we = __shfl_up_sync(0xffffffffu, wi, 1);
            const T tile_agg = __shfl_sync(0xffffffffu, wi, NWARPS - 1);
            if (lane < NWARPS) warp_exc[lane] = we;
            if (lane == 0) {
                if (p.protocol_checks) {
                    uint64_t w[S::W];
                    T dummy;
                    S::load(agg, t, w);
                    if (S::decode(w, tag, dummy)) raise_error(hdr, 5u /*LS_ERR_PROTOCOL*/, (uint32_t)t);
                }
                if (t != p.stall_tile || p.spin_budget <= 0)
                    S::publish(agg, t, tag, t == p.corrupt_tile ? ident : tile_agg);
            }
            T prefix = ident;
            const bool has = round_lookback<T, OP>(agg, rnd, k, c, G, tag, carry_in, lane, p.spin_budget, hdr,
                                                   prefix);
            const T incl = has ? OP::apply(prefix, tile_agg) : tile_agg;
            if (lane == 0) {
                if (c == G - 1 && t + 1 < M) S::publish(rnd, k, tag, incl);
                if (t == M - 1 && p.total_out != nullptr) *static_cast<T *>(p.total_out) = incl;
                *tile_pre = prefix;
                *tile_has = has ? 1 : 0;
            }
        }
        __syncthreads();  // (B)

        bool has = *tile_has != 0;
        T acc = *tile_pre;
        if (warp > 0) { acc = has ? OP::apply(acc, warp_exc[warp]) : warp_exc[warp]; has = true; }
        if (lane > 0) { acc = has ? OP::apply(acc, wexc) : wexc; has = true; }
#pragma unroll
        for (int i = 0; i < ITEMS; ++i) {
            const T v = r.e[i];
            const bool first = (i == 0 && !has);
            if (EXCL) {
                r.e[i] = first ? ident : acc;
                acc = first ? v : OP::apply(acc, v);
            } else {
                acc = first ? v : OP::apply(acc, v);
                r.e[i] = acc;
            }
        }
        store_tile_regs<T, V>(st, tid, r);
        __syncthreads();
        for (int i = tid; i < valid; i += THREADS) y[t0 + i] = sv[i];
        __syncthreads();  // the tile buffer is reused by the next iteration
    }
    __syncthreads();
    if (tid == 0) epoch_handover(hdr, tag, G);
}

template <typename T, int THREADS, int TILE_BYTES>
constexpr size_t scan_generic_smem_bytes() {
    return (size_t)TILE_BYTES + (size_t)(2 * (THREADS / 32) + 1) * sizeof(T) + 16;
}

// ------------------------------------------------------------------------------
// Deterministic grid reduction (the per-shard total for the multi-GPU carry
// exchange): thread-serial over a fixed grid-stride partition, fixed warp and
// block trees, the last CTA folds the per-CTA partials in index order.
// 256-bit loads, four in flight per thread (the read-only ceiling probe's
// access pattern, bench_support/copy_probe.cu).  The sweep runs from the end
// of x to its start, and the first keep_bytes of x — read last — are loaded
// evict-last: a carried scan of the same shard right behind it (the
// contiguous-shard step, distributed.sharded_scan) finds its first tiles in
// L2 instead of HBM.
template <typename T, typename OP, int THREADS>
__global__ void __launch_bounds__(THREADS) reduce_kernel(const T *__restrict__ x, int64_t n, T *total_out,
                                                         uint8_t *ws, int64_t keep_bytes) {
    constexpr int NWARPS = THREADS / 32;
    constexpr int PER = 32 / (int)sizeof(T);  // elements per 32-byte chunk
    __shared__ T wsum[NWARPS];
    __shared__ bool last;
    Header *hdr = reinterpret_cast<Header *>(ws);
    T *partials = reinterpret_cast<T *>(ws + sizeof(Header));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t gtid = (int64_t)blockIdx.x * THREADS + tid;
    const int64_t gstride = (int64_t)gridDim.x * THREADS;
    const T ident = OP::template identity<T>();

    const int64_t mis = (int64_t)(((uintptr_t)x & 31u) / sizeof(T));
    int64_t head = mis ? (PER - mis) : 0;
    if (head > n) head = n;
    const int64_t nch = (n - head) / PER;
    const int64_t tail0 = head + nch * PER;
    T acc = ident;
    if (gtid < head) acc = x[gtid];
    const uint8_t *xc = reinterpret_cast<const uint8_t *>(x + head);
    const uint64_t pol_first = policy_evict_first(), pol_last = policy_evict_last();
    const int64_t keep_ch = keep_bytes / 32;  // chunks [0, keep_ch): evict-last
    int64_t i = gtid;
    for (; i + 3 * gstride < nch; i += 4 * gstride) {
        Regs<T, 8> q;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int64_t v = nch - 1 - (i + u * gstride);  // reverse sweep
            ldg256_hint(xc + v * 32, q.q[2 * u], q.q[2 * u + 1], v < keep_ch ? pol_last : pol_first);
        }
#pragma unroll
        for (int j = 0; j < 4 * PER; ++j) acc = OP::apply(acc, q.e[j]);
    }
    for (; i < nch; i += gstride) {
        Regs<T, 2> q;
        const int64_t v = nch - 1 - i;
        ldg256_hint(xc + v * 32, q.q[0], q.q[1], v < keep_ch ? pol_last : pol_first);
#pragma unroll
        for (int j = 0; j < PER; ++j) acc = OP::apply(acc, q.e[j]);
    }
    if (gtid < n - tail0) acc = OP::apply(acc, x[tail0 + gtid]);

    acc = warp_reduce_fixed<T, OP>(acc);
    if (lane == 0) wsum[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        T v = lane < NWARPS ? wsum[lane] : ident;
        v = warp_reduce_fixed<T, OP>(v);
        if (lane == 0) {
            partials[blockIdx.x] = v;
            __threadfence();
            const uint32_t old = atom_add_acqrel_u32(&hdr->done, 1u);
            last = (old == gridDim.x - 1u);
        }
    }
    __syncthreads();
    if (last && warp == 0) {
        __threadfence();
        T v = ident;
        for (int b = lane; b < (int)gridDim.x; b += 32) v = OP::apply(v, *((volatile T *)&partials[b]));
        v = warp_reduce_fixed<T, OP>(v);
        if (lane == 0) {
            *total_out = v;
            if constexpr (order_sensitive<T, OP>())  // reduce_ties_kernel's search word
                *reinterpret_cast<long long *>(&hdr->pad[2]) = v != v ? 0x7fffffffffffffffll : -1ll;
            st_relaxed_u32(&hdr->done, 0u);
        }
    }
}

// Order-sensitive operators (float max/min): the reduction above combines out
// of sequence order, exact except for the bits of a zero or NaN total.  For
// those this kernel (launched right behind it) finds the element the
// sequential fold returns — the rightmost zero, or the leftmost NaN — and
// writes it as the total; otherwise every block returns at once.
template <typename T, typename OP, int THREADS>
__global__ void __launch_bounds__(THREADS) reduce_ties_kernel(const T *__restrict__ x, int64_t n, T *total_out,
                                                              uint8_t *ws) {
    __shared__ bool last;
    Header *hdr = reinterpret_cast<Header *>(ws);
    long long *best_word = reinterpret_cast<long long *>(&hdr->pad[2]);
    const T a = *total_out;
    if (!tie_class(a)) return;
    const bool nan = a != a;
    long long best = nan ? 0x7fffffffffffffffll : -1ll;
    for (int64_t i = (int64_t)blockIdx.x * THREADS + threadIdx.x; i < n; i += (int64_t)gridDim.x * THREADS) {
        const T v = x[i];
        if (nan ? v != v : v == (T)0) best = nan ? min(best, (long long)i) : max(best, (long long)i);
    }
    if (nan ? best != 0x7fffffffffffffffll : best >= 0) {
        if (nan) atomicMin(best_word, best);
        else atomicMax(best_word, best);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atom_add_acqrel_u32(&hdr->done, 1u) == gridDim.x - 1u;
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        *total_out = x[*(volatile long long *)best_word];
        st_relaxed_u32(&hdr->done, 0u);
    }
}

// carry_out = totals[0] (+) ... (+) totals[rank-1]  (fixed left fold)
template <typename T, typename OP>
__global__ void carry_kernel(const T *totals, int64_t rank, T *carry_out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        T acc = OP::template identity<T>();
        if (rank > 0) acc = totals[0];
        for (int64_t g = 1; g < rank; ++g) acc = OP::apply(acc, totals[g]);
        *carry_out = acc;
    }
}

}  // namespace lscan

namespace lscan {

// ------------------------------------------------------------------------------
// Slot handshake stress (the device analogue of the reference's C4,
// test_acceptance.py:146-196 / test_chained.py:287-323): one writer thread
// publishes `count` fresh slots in order with known values while reader warps
// chase it, each re-reading its own window of 64 slots until the writer is done
// (plus one final pass).  A reader that sees a slot's tag must see exactly the
// written value (no torn pair: for 64-bit T the two tagged halves), and a slot
// once seen published must stay published for that reader (flags monotone).
// stats[0] = reads, stats[1] = torn, stats[2] = regressions.
__device__ __forceinline__ uint64_t stress_value(int64_t i) {
    return ((uint64_t)i * 2654435761ull) & ((1ull << 62) - 1);
}

template <typename T>
__global__ void slot_stress_kernel(uint64_t *slots, int64_t count, uint32_t tag, volatile int *writer_done,
                                   unsigned long long *stats) {
    using S = Slot<T>;
    if (blockIdx.x == 0) {
        if (threadIdx.x == 0) {
            for (int64_t i = 0; i < count; ++i) {
                S::publish(slots, i, tag, (T)stress_value(i));
                if ((i & 255) == 255) __nanosleep(200);
            }
            __threadfence();
            *writer_done = 1;
        }
        return;
    }
    const int64_t reader = (int64_t)(blockIdx.x - 1) * blockDim.x + threadIdx.x;
    const int64_t base = (reader * 64) % (count > 64 ? count - 64 : 1);
    uint64_t seen = 0;
    unsigned long long reads = 0, torn = 0, regress = 0;
    bool finishing = false;
    while (true) {
        if (*writer_done) finishing = true;
        for (int b = 0; b < 64; ++b) {
            uint64_t w[S::W];
            T v;
            S::load(slots, base + b, w);
            const bool valid = S::decode(w, tag, v);
            ++reads;
            if (valid) {
                if (v != (T)stress_value(base + b)) ++torn;
                seen |= 1ull << b;
            } else if (seen & (1ull << b)) {
                ++regress;
            }
        }
        if (finishing) break;
    }
    atomicAdd(&stats[0], reads);
    atomicAdd(&stats[1], torn);
    atomicAdd(&stats[2], regress);
}

}  // namespace lscan
