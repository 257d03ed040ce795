// lscan_cluster.cuh — the latency path (small and mid n): one tile per
// block, blocks grouped in thread-block clusters, the inter-block carry
// passed through distributed shared memory inside a cluster and through
// epoch-tagged global slots between clusters.
//
// The reference's chain (chained.py:153-172: block i waits for block i-1's
// inclusive value) becomes "every block needs the sum of the blocks before
// it".  Inside a cluster (up to 16 co-scheduled blocks) that exchange is one
// DSMEM store per (block, later block) pair and one cluster barrier.  Across
// clusters each cluster publishes its aggregate as soon as its barrier
// passes — it depends on nothing outside the cluster — and every block folds
// the aggregates of the clusters before it: one L2 round trip, no serial
// chain.  All clusters are co-resident (cooperative launch), so the waits
// cannot deadlock.  With one cluster there are no slots and no epoch at all:
// launch + one load + the block scan + one cluster barrier + one store.
//
// Block b owns tile b (TILE_ELEMS contiguous elements).  Inside
// the block the layout and the scan are the hot kernel's (Alg. 2/3/5,
// warp.py:85-169): each warp owns WARP_BYTES contiguous bytes as V rows of
// 32 lanes x 16-byte vectors; per row a thread-serial fold, a
// __shfl_up_sync warp scan and a serial row carry; a shared-memory scan of
// the warp totals; the carry folded in registers and stored with 128-bit
// stores.  Any element-aligned x / y works: vectors that are misaligned or
// cross the end of the array fall back to element accesses.
#pragma once
#include "lscan_common.cuh"

namespace lscan {

// lab: per-block event times (%globaltimer ns) into the buffer p.xchg points
// at (bench_support/cluster_lab.cu builds with -DLS_LAB_CTIMELINE=1; the
// product never sets p.xchg for this kernel): [b][0] start, [1] loads + row
// scans done, [2] cluster exchange done, [3] block prefix known, [4] stores
// issued, [5] warp 0's DSMEM stores issued — held in registers and written
// at the very end (a global store before the cluster barrier's release would
// delay it) — scripts/cluster_timeline.py
#ifndef LS_LAB_CTIMELINE
#define LS_LAB_CTIMELINE 0
#endif
constexpr int kCTimelineWords = 6;

// Lab (LS_CLUSTER_EARLY_AGG=1): with several clusters, the last block of each
// cluster publishes the cluster aggregate as soon as the other blocks'
// aggregates have landed in its shared memory (each storer arrives on an
// mbarrier there, release at cluster scope) instead of after the cluster
// barrier.  Measured slower: i64 2^17 4.33 -> 5.27 us, 2^20 7.10 -> 8.22,
// i32 2^21 6.82 -> 7.25 (profiles/r2_cluster_early_agg_ab.jsonl); off
#ifndef LS_CLUSTER_EARLY_AGG
#define LS_CLUSTER_EARLY_AGG 0
#endif

__device__ __forceinline__ void mbar_arrive_remote_cluster(uint32_t remote_bar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_wait_acquire_cluster(uint64_t *bar, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
    } while (!ok);
}


__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// address of `local` (this CTA's shared memory) in CTA `cta` of the cluster
__device__ __forceinline__ uint32_t mapa_shared(uint32_t local, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(cta));
    return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_u64(uint32_t addr, uint64_t v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
// split cluster barrier (every thread of every CTA): the first phase only
// guarantees every CTA of the cluster has started before anyone stores into
// its shared memory, so it is relaxed and its latency hides behind the loads
__device__ __forceinline__ void cluster_arrive_relaxed() {
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.aligned;" ::: "memory"); }
// every thread of every CTA of the cluster; release/acquire orders the DSMEM
// stores issued before the arrival with the loads after the wait
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ void stg128_v4(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ uint4 ldg128(const void *p) {
    uint4 v;
    asm volatile("ld.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
    return v;
}

// VW: 16-byte vectors per lane per row (1, or 2 for 32-byte lane chunks moved
// by 256-bit accesses: half the warp scans per element)
template <typename T, typename OP, bool EXCL, int V, int THREADS, int MINB, int VW = 1>
__global__ void __launch_bounds__(THREADS, MINB) scan_cluster_kernel(const ScanParams p) {
    constexpr int WARPS = THREADS / 32;
    constexpr int PER = 16 / (int)sizeof(T);
    constexpr int WARP_VECS = 32 * V;
    constexpr int TILE_ELEMS = WARPS * WARP_VECS * PER;
    constexpr int VR = V / VW;       // rows per lane
    constexpr int RPER = VW * PER;   // elements per lane per row
    static_assert(V % VW == 0 && (VW == 1 || VW == 2), "rows of one or two vectors per lane");
    using Bits = typename Elem<T>::Bits;
    using S = Slot<T>;

    __shared__ T warp_tot[WARPS];
    __shared__ T warp_exc[WARPS];
    __shared__ T row_tot[WARPS][VR];      // per warp: totals of its rows
    __shared__ Bits cta_agg[kClusterMax];  // aggregates of the lower blocks of this cluster, stored by them
    __shared__ T block_agg;
    __shared__ T s_pre;                    // carry (+) clusters before this one (+) blocks before this one
    __shared__ int s_has;
    __shared__ __align__(8) uint64_t agg_bar;  // last block: the other blocks' aggregates have landed

    // programmatic dependent launch: the grid may start while the previous
    // kernel in the stream drains; nothing global is touched before this wait
    // (which returns once that kernel has completed and flushed), and the
    // next kernel may begin launching as soon as every block got here
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint64_t tl_t[kCTimelineWords] = {};
    auto tl_mark = [&](int idx) {  // LS_LAB_CTIMELINE only
        if constexpr (LS_LAB_CTIMELINE) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tl_t[idx]));
    };
    tl_mark(0);
    const uint32_t r = cluster_ctarank();
    const uint32_t C = cluster_nctarank();
    const int64_t b = blockIdx.x;        // tile index
    const int64_t k = b / C;             // cluster index
    const int64_t K = gridDim.x / C;     // clusters in the grid
    // (not for float max / min: the extra fold's registers spilled the f64 forms)
    const bool early_agg = LS_CLUSTER_EARLY_AGG && !order_sensitive<T, OP>() && K > 1 && C > 1;
    if (early_agg && r == C - 1 && tid == 0) {
        mbar_init(&agg_bar, C - 1);
        fence_mbar_init();  // visible cluster-wide before the phase-1 barrier completes
    }
    if (C > 1) cluster_arrive_relaxed();  // phase 1: "this CTA is running" (waited on before DSMEM stores)
    const T ident = OP::template identity<T>();
    const int64_t t0 = b * TILE_ELEMS;
    int64_t valid = p.n - t0 < TILE_ELEMS ? p.n - t0 : TILE_ELEMS;  // <= 0: a padding block of the last cluster
    if (valid < 0) valid = 0;
    const T *x = static_cast<const T *>(p.x) + t0;
    T *y = static_cast<T *>(p.y) + t0;
    const bool xv = ((uintptr_t)x & 15u) == 0, yv = ((uintptr_t)y & 15u) == 0;
    const bool xw = ((uintptr_t)x & 31u) == 0, yw = ((uintptr_t)y & 31u) == 0;  // 256-bit capable
    Header *hdr = reinterpret_cast<Header *>(p.ws);
    const uint32_t tag = K > 1 ? call_tag(hdr) : 0u;

    // ---- load: row j of warp w is vectors w*WARP_VECS + (j*32 + lane)*VW + u.
    //      Whole aligned tiles take a branch-free path so all loads are in
    //      flight at once (a per-row branch makes the compiler wait on each).
    Regs<T, V> d;
    if (xv && valid == TILE_ELEMS) {
#pragma unroll
        for (int j = 0; j < VR; ++j) {
            const T *src = x + (int64_t)(warp * WARP_VECS + (j * 32 + lane) * VW) * PER;
            if (VW == 2 && xw) ldg256(src, d.q[2 * j], d.q[2 * j + 1]);
            else
#pragma unroll
                for (int u = 0; u < VW; ++u) d.q[j * VW + u] = ldg128(src + u * PER);
        }
    } else {
#pragma unroll
        for (int j = 0; j < VR; ++j) {
#pragma unroll
            for (int u = 0; u < VW; ++u) {
                const int64_t e0 = (int64_t)(warp * WARP_VECS + (j * 32 + lane) * VW + u) * PER;
                if (xv && e0 + PER <= valid) {
                    d.q[j * VW + u] = ldg128(x + e0);
                } else {
#pragma unroll
                    for (int e = 0; e < PER; ++e) d.e[(j * VW + u) * PER + e] = e0 + e < valid ? x[e0 + e] : ident;
                }
            }
        }
    }

    // ---- per row: lane-serial fold of the vector and an inclusive warp scan,
    //      then the serial row carry (Alg. 2)
    //      (row totals go to shared memory: registers are kept for the tile)
    T rex[VR];
    T run = ident;
#pragma unroll
    for (int j = 0; j < VR; ++j) {
        T v = d.e[j * RPER];
#pragma unroll
        for (int e = 1; e < RPER; ++e) v = OP::apply(v, d.e[j * RPER + e]);
        const T inc = warp_inclusive_scan<T, OP, true>(v, lane);
        if constexpr (std::is_integral<T>::value && OP::code == OpAdd::code)
            rex[j] = OP::apply(inc, (T)(0 - (typename std::make_unsigned<T>::type)v));  // inc - v, exact
        else
            rex[j] = __shfl_up_sync(0xffffffffu, inc, 1);
        const T rt = __shfl_sync(0xffffffffu, inc, 31);
        if (lane == 0) row_tot[warp][j] = rt;
        run = j == 0 ? rt : OP::apply(run, rt);
    }
    if (lane == 0) warp_tot[warp] = run;
    if (C > 1) cluster_wait();  // every CTA of the cluster has started: its shared memory may be written
    __syncthreads();
    tl_mark(1);

    // the earlier clusters' aggregates, folded in cluster order (warp 0)
    uint64_t *const slots = reinterpret_cast<uint64_t *>(p.ws + kSlotBase);
    auto read_prev = [&]() -> T {
        T acc = ident;
        for (int64_t base = 0; base < k; base += 32) {
            const int64_t j = base + lane;
            T v = ident;
            if (j < k) {
                uint64_t w[S::W];
                S::load(slots, j, w);
                while (!S::decode(w, tag, v)) {
                    __nanosleep(20);
                    S::load(slots, j, w);
                }
            }
            acc = fold_chunk<T, OP>(acc, v);
        }
        return fold_finish<T, OP>(acc);
    };

    // ---- warp totals -> exclusive warp prefixes; the block aggregate goes to
    //      every later block of the cluster (DSMEM), slot r
    if (warp == 0) {
        const T wi = warp_inclusive_scan<T, OP, true>(lane < WARPS ? warp_tot[lane] : ident, lane);
        const T we = __shfl_up_sync(0xffffffffu, wi, 1);
        if (lane < WARPS) warp_exc[lane] = we;
        const T agg = __shfl_sync(0xffffffffu, wi, WARPS - 1);
        const uint32_t local = smem_u32(&cta_agg[r]);
        for (uint32_t q = r + 1 + (uint32_t)lane; q < C; q += 32) {
            const uint32_t a = mapa_shared(local, q);
            if constexpr (sizeof(T) == 4) st_cluster_u32(a, Elem<T>::bits(agg));
            else st_cluster_u64(a, Elem<T>::bits(agg));
            // the store into the last block, then (release, cluster scope) its arrival
            if (early_agg && q == C - 1) mbar_arrive_remote_cluster(mapa_shared(smem_u32(&agg_bar), q));
        }
        if (lane == 0) block_agg = agg;
        if (early_agg && r == C - 1 && lane == 0) {
            // every other block's aggregate is here: publish the cluster's at once
            // (the same left fold the blocks of the next clusters expect)
            mbar_wait_acquire_cluster(&agg_bar, 0u);
            T pc = Elem<T>::from(cta_agg[0]);
            for (uint32_t q = 1; q < r; ++q) pc = OP::apply(pc, Elem<T>::from(cta_agg[q]));
            S::publish(slots, k, tag, OP::apply(pc, agg));
        }
        tl_mark(5);
    }
    if (C > 1) cluster_sync_all();
    else __syncthreads();
    tl_mark(2);

    // ---- block prefix = carry (+) [clusters 0..k-1] (+) [blocks 0..r-1 of this cluster]
    if (warp == 0) {
        // in-cluster part, fixed order
        bool hc = false;
        T pc = ident;
        for (uint32_t q = 0; q < r; ++q) {
            const T a = Elem<T>::from(cta_agg[q]);
            pc = hc ? OP::apply(pc, a) : a;
            hc = true;
        }
        bool has = p.carry_in != nullptr;
        T pre = has ? *static_cast<const T *>(p.carry_in) : ident;
        if (K > 1) {
            // the cluster's aggregate depends on nothing outside the cluster:
            // published at once, so the wait below is one L2 round trip, not
            // a chain (clusters are co-resident: cooperative launch)
            if (!early_agg && r == C - 1 && lane == 0)
                S::publish(slots, k, tag, hc ? OP::apply(pc, block_agg) : block_agg);
            if (k > 0) {
                const T g = read_prev();
                pre = has ? OP::apply(pre, g) : g;
                has = true;
            }
        }
        if (r > 0) {
            pre = has ? OP::apply(pre, pc) : pc;
            has = true;
        }
        if (lane == 0) {
            s_pre = pre;
            s_has = has ? 1 : 0;
            if (p.total_out != nullptr && valid > 0 && t0 + valid == p.n)
                *static_cast<T *>(p.total_out) = has ? OP::apply(pre, block_agg) : block_agg;
        }
    }
    __syncthreads();
    tl_mark(3);
    bool has0 = s_has != 0;
    T pre = s_pre;
    if (warp > 0) {
        pre = has0 ? OP::apply(pre, warp_exc[warp]) : warp_exc[warp];
        has0 = true;
    }

    // ---- fold the carry in registers, store; rowpre = rows before j (the
    //      serial row carry, rebuilt here to keep registers for large tiles)
    T rowpre = row_tot[warp][0];
#pragma unroll
    for (int j = 0; j < VR; ++j) {
        bool has = has0;
        T acc = pre;
        if (j > 0) {
            acc = has ? OP::apply(acc, rowpre) : rowpre;
            has = true;
            if (j + 1 < VR) rowpre = OP::apply(rowpre, row_tot[warp][j]);
        }
        if (lane > 0) { acc = has ? OP::apply(acc, rex[j]) : rex[j]; has = true; }
#pragma unroll
        for (int e = 0; e < RPER; ++e) {
            const T v = d.e[j * RPER + e];
            const bool first = (e == 0 && !has);
            if (EXCL) {
                d.e[j * RPER + e] = first ? ident : acc;
                acc = first ? v : OP::apply(acc, v);
            } else {
                acc = first ? v : OP::apply(acc, v);
                d.e[j * RPER + e] = acc;
            }
        }
    }
    if (yv && valid == TILE_ELEMS) {
#pragma unroll
        for (int j = 0; j < VR; ++j) {
            T *dst = y + (int64_t)(warp * WARP_VECS + (j * 32 + lane) * VW) * PER;
            if (VW == 2 && yw) stg256(dst, d.q[2 * j], d.q[2 * j + 1]);
            else
#pragma unroll
                for (int u = 0; u < VW; ++u) stg128_v4(dst + u * PER, d.q[j * VW + u]);
        }
    } else {
#pragma unroll
        for (int j = 0; j < VR; ++j) {
#pragma unroll
            for (int u = 0; u < VW; ++u) {
                const int64_t e0 = (int64_t)(warp * WARP_VECS + (j * 32 + lane) * VW + u) * PER;
                if (yv && e0 + PER <= valid) {
                    stg128_v4(y + e0, d.q[j * VW + u]);
                } else {
#pragma unroll
                    for (int e = 0; e < PER; ++e)
                        if (e0 + e < valid) y[e0 + e] = d.e[(j * VW + u) * PER + e];
                }
            }
        }
    }
    tl_mark(4);
    if (LS_LAB_CTIMELINE && p.xchg != nullptr && tid == 0)
        for (int i = 0; i < kCTimelineWords; ++i)
            reinterpret_cast<uint64_t *>(p.xchg)[(int64_t)blockIdx.x * kCTimelineWords + i] = tl_t[i];
    // the last block to finish records this call's tag as the workspace epoch
    // (relaxed: nothing in this grid reads the epoch again, and the next call
    // starts after this grid has completed)
    if (K > 1 && tid == 0) {
        if (atomicAdd(&hdr->done, 1u) == gridDim.x - 1u) {
            st_relaxed_u32(&hdr->done, 0u);
            st_relaxed_u32(&hdr->epoch, tag);
        }
    }
}


}  // namespace lscan
