// lscan_scan_ws.cuh — the warp-specialised persistent scan (the hot path).
//
// Same algorithm and slot protocol as scan_kernel (lscan_kernels.cuh: round
// look-back over epoch-tagged aggregate slots A[t] and round prefixes R[r]),
// but the roles the reference's worker performs in sequence
// (chained.py:237-249: local accumulate -> inter_block_comm -> combine) run
// as concurrent warp roles inside each persistent CTA, so the cross-CTA
// carry chain is resolved AHEAD of the data pass instead of stalling it:
//
//   producer warp   TMA bulk loads of x tiles into a STAGES-deep smem ring,
//                   TMA bulk stores of finished tiles to y, stage recycling
//   reducer warp    sums each tile as soon as it lands and publishes A[t]
//                   (never waits on another CTA)
//   look-back warp  prefix(t) = R[r-1] (+) A[rG] (+) ... (+) A[rG+c-1] into a
//                   smem ring; in CTA G-1 it also publishes R[r] = prefix + A[t]
//                   (the only serial chain: one L2 round trip per round)
//   scanner warps   register tile -> thread-serial + warp-shuffle + smem scan,
//                   fold in prefix(t), write back to the stage for the store
//
// Measured motivation (profiles/r1_lab_v1_lookback_vs_nolookback.json): the
// sequential kernel moves data at 6.2-6.7 TB/s when the look-back is skipped
// but only ~3.3 TB/s with it — the chain, not the data path, was the limit.
#pragma once
#include "lscan_kernels.cuh"

namespace lscan {

template <typename T, int TILE_BYTES>
__device__ __forceinline__ T reduce_stage(const uint8_t *st, int lane) {
    constexpr int NV = TILE_BYTES / 16 / 32;  // 16-byte vectors per lane
    constexpr int PER = 16 / (int)sizeof(T);
    static_assert(NV % 4 == 0, "tile must hold a multiple of 4 vectors per lane");
    T acc[4] = {T(0), T(0), T(0), T(0)};
    const uint32_t base = smem_u32(st) + (uint32_t)lane * 16;
#pragma unroll 2
    for (int j = 0; j < NV; j += 4) {
        Regs<T, 4> r;
#pragma unroll
        for (int u = 0; u < 4; ++u) r.q[u] = lds128(base + (uint32_t)(j + u) * 512u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[u] = acc[u] + r.e[u * PER + e];
    }
    return warp_sum_fixed((acc[0] + acc[1]) + (acc[2] + acc[3]));
}

// One look-back step of the aux warp for tile t = k*G + c, all loads in
// flight at once: the round prefix R[k-1] (when need_r), the aggregates
// A[kG .. kG+c-1] and, when want_own, A[t] itself.  Spins until every word
// carries `tag`.  Sums are fixed-order (lane-serial ascending, butterfly), so
// the result does not depend on timing.
template <typename T>
struct LookbackOut {
    T r;     // R[k-1]
    T sum;   // A[kG] (+) ... (+) A[kG+c-1]
    T own;   // A[t]
};

template <typename T>
__device__ __forceinline__ LookbackOut<T> aux_lookback(const uint64_t *agg, const uint64_t *rnd, int64_t k, int c,
                                                       int G, bool need_r, bool want_own, uint32_t tag, int lane,
                                                       int64_t spin_budget, Header *hdr, uint32_t where) {
    using S = Slot<T>;
    constexpr int U = 5;  // 160 slots per pass covers a 148-SM round
    const int count = c + (want_own ? 1 : 0);
    const int64_t first = k * (int64_t)G;
    T acc = T(0), own = T(0), r = T(0);
    int64_t probes = 0;
    bool r_pending = need_r;
    uint64_t rw[S::W];
    if (need_r) S::load(rnd, k - 1, rw);
    for (int base = 0; base < count || r_pending; base += 32 * U) {
        uint64_t w[U][S::W];
        bool need[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * 32 + lane;
            need[u] = j < count;
            if (need[u]) S::load(agg, first + j, w[u]);
        }
        T val[U];
        while (true) {
            bool ok = true;
            if (r_pending) {
                if (S::decode(rw, tag, r)) r_pending = false;
                else ok = false;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (need[u]) {
                    if (S::decode(w[u], tag, val[u])) need[u] = false;
                    else ok = false;
                }
            }
            if (__all_sync(0xffffffffu, ok)) break;
            if (spin_budget > 0 && ++probes > spin_budget) {
                if (lane == 0) raise_error(hdr, 4u /*LS_ERR_LIVENESS*/, where);
                if (r_pending) { r = T(0); r_pending = false; }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (need[u]) { val[u] = T(0); need[u] = false; }
                break;
            }
            __nanosleep(32);
            if (r_pending) S::load(rnd, k - 1, rw);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = base + u * 32 + lane;
                if (need[u]) S::load(agg, first + j, w[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * 32 + lane;
            if (j < c) acc = acc + val[u];
            else if (j == c && want_own) own = val[u];
        }
    }
    LookbackOut<T> o;
    o.sum = warp_sum_fixed(acc);
    o.r = r;
    o.own = want_own ? __shfl_sync(0xffffffffu, own, c & 31) : T(0);
    return o;
}

template <typename T, int SCAN_WARPS, int TILE_BYTES, int STAGES, bool EXCL>
__global__ void __launch_bounds__((SCAN_WARPS + 3) * 32, 1) scan_ws_kernel(const ScanParams p) {
    constexpr int SCAN_THREADS = SCAN_WARPS * 32;
    constexpr int V = TILE_BYTES / SCAN_THREADS / 16;
    constexpr int ITEMS = V * 16 / (int)sizeof(T);
    constexpr int TILE_ELEMS = TILE_BYTES / (int)sizeof(T);
    constexpr int W_PROD = SCAN_WARPS, W_RED = SCAN_WARPS + 1, W_AUX = SCAN_WARPS + 2;
    static_assert(V >= 1 && (V & (V - 1)) == 0, "vectors per thread must be a power of two");
    static_assert(SCAN_WARPS >= 2 && SCAN_WARPS <= 32, "2..32 scanner warps");
    using S = Slot<T>;

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *stages = smem;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * TILE_BYTES);  // data landed
    uint64_t *red_done = full + STAGES;                                         // reducer finished reading
    uint64_t *res_ready = red_done + STAGES;                                    // results in the stage
    uint64_t *pre_ready = res_ready + STAGES;                                   // prefix in pre[]
    T *pre = reinterpret_cast<T *>(pre_ready + STAGES);                         // [STAGES]
    int *pre_has = reinterpret_cast<int *>(pre + STAGES);                       // [STAGES]
    T *warp_tot = reinterpret_cast<T *>(pre_has + STAGES + (STAGES & 1));       // [SCAN_WARPS]
    T *warp_exc = warp_tot + SCAN_WARPS;                                        // [SCAN_WARPS]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t M = p.num_tiles;
    Header *hdr = reinterpret_cast<Header *>(p.ws);
    uint64_t *agg = reinterpret_cast<uint64_t *>(p.ws + kSlotBase);
    uint64_t *rnd = agg + M * S::W;
    const T *x = static_cast<const T *>(p.x);
    T *y = static_cast<T *>(p.y);

    const uint32_t prev_epoch = ld_relaxed_u32(&hdr->epoch);
    const uint32_t tag = (prev_epoch + 1u) == 0u ? 1u : prev_epoch + 1u;
    const int64_t my_tiles = (M - c + G - 1) / G;
    const int64_t full_tiles = p.n / TILE_ELEMS;

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&red_done[s], 1);
            mbar_init(&res_ready[s], 1);
            mbar_init(&pre_ready[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();

    if (warp == W_PROD) {
        // ------------------------------------------------------------ producer
        const uint64_t pol = policy_evict_first();
        auto load_tile = [&](int64_t k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            const int64_t t0 = t * TILE_ELEMS;
            if (t < full_tiles) {
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[s], TILE_BYTES);
                    tma_load_1d(stages + s * TILE_BYTES, x + t0, TILE_BYTES, &full[s], pol);
                }
            } else {
                // partial_tail (chained.py:188-202): identity-padded last tile
                const int64_t valid = p.n - t0;
                T *sv = reinterpret_cast<T *>(stages + s * TILE_BYTES);
                for (int i = lane; i < TILE_ELEMS; i += 32) sv[i] = (i < valid) ? x[t0 + i] : T(0);
                __syncwarp();
                if (lane == 0) mbar_arrive(&full[s]);
            }
        };
        for (int64_t k = 0; k < STAGES && k < my_tiles; ++k) load_tile(k);
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            const int64_t t0 = t * TILE_ELEMS;
            mbar_wait(&res_ready[s], (uint32_t)((k / STAGES) & 1));
            if (t < full_tiles) {
                if (lane == 0) {
                    tma_store_1d(y + t0, stages + s * TILE_BYTES, TILE_BYTES, pol);
                    bulk_commit();
                }
            } else {
                const int64_t valid = p.n - t0;
                const T *sv = reinterpret_cast<const T *>(stages + s * TILE_BYTES);
                for (int i = lane; i < valid; i += 32) y[t0 + i] = sv[i];
            }
            // recycle the previous tile's stage for the tile STAGES ahead of it
            const int64_t kn = k - 1 + STAGES;
            if (k >= 1 && kn < my_tiles) {
                const int sp = (int)((k - 1) % STAGES);
                if (lane == 0) bulk_wait_read<1>();
                mbar_wait(&red_done[sp], (uint32_t)(((k - 1) / STAGES) & 1));
                __syncwarp();
                load_tile(kn);
            }
        }
        if (lane == 0) bulk_wait_all();
    } else if (warp == W_RED) {
        // ------------------------------------------------------------- reducer
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
            if (p.delay_red_ns > 0 && t % 3 == 1) debug_sleep(p.delay_red_ns);
            const T a = reduce_stage<T, TILE_BYTES>(stages + s * TILE_BYTES, lane);
            __syncwarp();
            if (lane == 0) {
                if (p.protocol_checks) {
                    uint64_t w[S::W];
                    T dummy;
                    S::load(agg, t, w);
                    if (S::decode(w, tag, dummy)) raise_error(hdr, 5u /*LS_ERR_PROTOCOL*/, (uint32_t)t);
                }
                if (t != p.stall_tile || p.spin_budget <= 0) S::publish(agg, t, tag, t == p.corrupt_tile ? T(0) : a);
                mbar_arrive(&red_done[s]);
            }
        }
    } else if (warp == W_AUX) {
        // ----------------------------------------------------------- look-back
        const T *carry_in = static_cast<const T *>(p.carry_in);
        const bool have_carry = carry_in != nullptr;
        T r_prev = have_carry ? *carry_in : T(0);  // R[k-1] as known to CTA G-1 (the chain owner)
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            const bool chain = (c == G - 1) && (t + 1 < M);
            // R[k-1]: the caller's carry in round 0, the chain owner's register,
            // or the published round slot for everyone else
            const bool need_r = k > 0 && c != G - 1;
            const LookbackOut<T> lb = aux_lookback<T>(agg, rnd, k, c, G, need_r, chain, tag, lane, p.spin_budget,
                                                      hdr, (uint32_t)t);
            bool has;
            T base;
            if (k == 0) { has = have_carry; base = r_prev; }
            else if (c == G - 1) { has = true; base = r_prev; }
            else { has = true; base = lb.r; }
            T prefix = base;
            if (c > 0) {
                prefix = has ? (base + lb.sum) : lb.sum;
                has = true;
            }
            if (chain) {
                // the chain: R[k] = prefix(t) (+) A[t]
                r_prev = has ? (prefix + lb.own) : lb.own;
                if (lane == 0) S::publish(rnd, k, tag, r_prev);
            }
            if (k >= STAGES) mbar_wait(&res_ready[s], (uint32_t)(((k - STAGES) / STAGES) & 1));
            if (lane == 0) {
                pre[s] = prefix;
                pre_has[s] = has ? 1 : 0;
                mbar_arrive(&pre_ready[s]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ scanners
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const uint32_t parity = (uint32_t)((k / STAGES) & 1);
            const int64_t t = c + k * G;
            uint8_t *st = stages + s * TILE_BYTES;
            mbar_wait(&full[s], parity);
            if (p.delay_scan_ns > 0 && t % 3 == 2 && warp == (int)(t % SCAN_WARPS)) debug_sleep(p.delay_scan_ns);
            Regs<T, V> r;
            load_tile_regs<T, V>(st, tid, r);
            T tsum = r.e[0];
#pragma unroll
            for (int i = 1; i < ITEMS; ++i) tsum = tsum + r.e[i];
            const T winc = warp_inclusive_scan(tsum, lane);
            const T wexc = __shfl_up_sync(0xffffffffu, winc, 1);
            if (lane == 31) warp_tot[warp] = winc;
            named_bar_sync(1, SCAN_THREADS);  // (A)
            if (warp == 0) {
                const T wt = lane < SCAN_WARPS ? warp_tot[lane] : T(0);
                const T wi = warp_inclusive_scan(wt, lane);
                const T we = __shfl_up_sync(0xffffffffu, wi, 1);
                if (lane < SCAN_WARPS) warp_exc[lane] = we;
            }
            mbar_wait(&pre_ready[s], parity);
            named_bar_sync(1, SCAN_THREADS);  // (B)
            bool has = pre_has[s] != 0;
            T acc = pre[s];
            if (warp > 0) { acc = has ? (acc + warp_exc[warp]) : warp_exc[warp]; has = true; }
            if (lane > 0) { acc = has ? (acc + wexc) : wexc; has = true; }
            if (EXCL) {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    const T v = r.e[i];
                    r.e[i] = (i == 0 && !has) ? T(0) : acc;
                    acc = (i == 0 && !has) ? v : (acc + v);
                }
            } else {
#pragma unroll
                for (int i = 0; i < ITEMS; ++i) {
                    acc = (i == 0 && !has) ? r.e[0] : (acc + r.e[i]);
                    r.e[i] = acc;
                }
            }
            if (t == M - 1 && tid == SCAN_THREADS - 1 && p.total_out != nullptr)
                *static_cast<T *>(p.total_out) = acc;
            // the results overwrite the stage in place: the reducer must be done
            // reading it (it usually is — it runs ahead — but CTAs whose prefix
            // does not depend on their own aggregate can get here first)
            mbar_wait(&red_done[s], parity);
            store_tile_regs<T, V>(st, tid, r);
            fence_proxy_async_smem();
            named_bar_sync(1, SCAN_THREADS);  // (C)
            if (tid == 0) mbar_arrive(&res_ready[s]);
        }
    }

    __syncthreads();
    if (tid == 0) {
        const uint32_t old = atom_add_acqrel_u32(&hdr->done, 1u);
        if (old == (uint32_t)G - 1u) {
            st_relaxed_u32(&hdr->done, 0u);
            st_relaxed_u32(&hdr->epoch, tag);
        }
    }
}

template <typename T, int SCAN_WARPS, int TILE_BYTES, int STAGES>
constexpr size_t scan_ws_smem_bytes() {
    return (size_t)STAGES * TILE_BYTES + 4 * STAGES * 8 + STAGES * sizeof(T) + (STAGES + 1) * 4 +
           2 * SCAN_WARPS * sizeof(T) + 32;
}

}  // namespace lscan
