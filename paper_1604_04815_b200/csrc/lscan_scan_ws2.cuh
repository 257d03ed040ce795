// lscan_scan_ws2.cuh — warp-specialised persistent scan, register-resident
// results (the hot path).
//
// Differs from scan_ws_kernel (lscan_scan_ws.cuh) in where a tile lives
// after it lands: the scanner warps copy it from the shared-memory stage
// into registers in the paper's lane-strided layout (Alg. 2,
// PAPER.md:137-189; warp.py:85-90 regs[j, i] = tile[i + W*j], here with
// 16-byte vectors as the "element" of a row) and release the stage at once,
// so the TMA ring holds only data in flight — not tiles waiting for their
// prefix.  Results go from registers straight to y with coalesced 128-bit
// stores (each warp instruction covers 512 contiguous bytes).
//
//   producer warp   TMA bulk loads into a STAGES-deep ring; a stage is
//                   refilled as soon as the scanners and the reducer have
//                   read it
//   reducer warp    sums each landed tile, publishes A[t] (never waits on
//                   another CTA)
//   look-back warp  prefix(t) = R[r-1] (+) A[rG..rG+c-1] into a smem ring;
//                   CTA G-1 also publishes R[r] (the only serial chain)
//   scanner warps   V rows per warp: thread-serial fold of each 16-byte
//                   vector, __shfl_up_sync row scan, serial row carry
//                   (Alg. 2), smem scan of warp totals (Alg. 3), prefix fold
//                   and store (Alg. 5)
#pragma once
#include "lscan_scan_ws.cuh"

namespace lscan {

__device__ __forceinline__ void stg128(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

template <typename T, int SCAN_WARPS, int TILE_BYTES, int STAGES, bool EXCL>
__global__ void __launch_bounds__((SCAN_WARPS + 3) * 32, 1) scan_ws2_kernel(const ScanParams p) {
    constexpr int SCAN_THREADS = SCAN_WARPS * 32;
    constexpr int V = TILE_BYTES / SCAN_THREADS / 16;  // rows (16-byte vectors) per lane
    constexpr int PER = 16 / (int)sizeof(T);           // elements per vector
    constexpr int TILE_ELEMS = TILE_BYTES / (int)sizeof(T);
    constexpr int WARP_BYTES = TILE_BYTES / SCAN_WARPS;
    constexpr int W_PROD = SCAN_WARPS, W_RED = SCAN_WARPS + 1, W_AUX = SCAN_WARPS + 2;
    static_assert(V >= 1, "at least one row per lane");
    static_assert(SCAN_WARPS >= 2 && SCAN_WARPS + 3 <= 32, "2..29 scanner warps");
    using S = Slot<T>;

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *stages = smem;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * TILE_BYTES);  // data landed
    uint64_t *empty = full + STAGES;      // scanners + reducer done reading (2 arrivals)
    uint64_t *pre_ready = empty + STAGES; // prefix written
    uint64_t *pre_free = pre_ready + STAGES;  // prefix consumed
    T *pre = reinterpret_cast<T *>(pre_free + STAGES);
    int *pre_has = reinterpret_cast<int *>(pre + STAGES);
    T *warp_tot = reinterpret_cast<T *>(pre_has + STAGES + (STAGES & 1));
    T *warp_exc = warp_tot + SCAN_WARPS;

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
            mbar_init(&empty[s], 2);
            mbar_init(&pre_ready[s], 1);
            mbar_init(&pre_free[s], 1);
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
                // partial_tail (chained.py:188-202): the 16-byte-aligned prefix of
                // the last tile by TMA, the ragged vector by plain loads, the rest
                // of the stage identity-filled with 128-bit shared stores
                const int64_t valid = p.n - t0;
                const uint32_t bulk = (uint32_t)((valid * (int64_t)sizeof(T)) & ~(int64_t)15);
                const int vfirst = (int)(bulk / 16);  // first vector not covered by TMA
                uint8_t *sb = stages + s * TILE_BYTES;
                const uint32_t sbase = smem_u32(sb);
                for (int v = vfirst + 1 + lane; v < TILE_BYTES / 16; v += 32) sts128(sbase + (uint32_t)v * 16u, make_uint4(0, 0, 0, 0));
                if (lane == 0 && vfirst < TILE_BYTES / 16) {
                    Regs<T, 1> rv;
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        const int64_t i = (int64_t)vfirst * PER + e;
                        rv.e[e] = i < valid ? x[t0 + i] : T(0);
                    }
                    sts128(sbase + (uint32_t)vfirst * 16u, rv.q[0]);
                }
                __syncwarp();
                if (lane == 0) {
                    if (bulk) {
                        mbar_arrive_expect_tx(&full[s], bulk);
                        tma_load_1d(sb, x + t0, bulk, &full[s], pol);
                    } else {
                        mbar_arrive(&full[s]);
                    }
                }
            }
        };
        for (int64_t k = 0; k < STAGES && k < my_tiles; ++k) load_tile(k);
        for (int64_t k = 0; k + STAGES < my_tiles; ++k) {
            mbar_wait(&empty[k % STAGES], (uint32_t)((k / STAGES) & 1));
            load_tile(k + STAGES);
        }
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
                mbar_arrive(&empty[s]);
                if (p.protocol_checks) {
                    uint64_t w[S::W];
                    T dummy;
                    S::load(agg, t, w);
                    if (S::decode(w, tag, dummy)) raise_error(hdr, 5u /*LS_ERR_PROTOCOL*/, (uint32_t)t);
                }
                if (t != p.stall_tile || p.spin_budget <= 0) S::publish(agg, t, tag, t == p.corrupt_tile ? T(0) : a);
            }
        }
    } else if (warp == W_AUX) {
        // ----------------------------------------------------------- look-back
        const T *carry_in = static_cast<const T *>(p.carry_in);
        const bool have_carry = carry_in != nullptr;
        T r_prev = have_carry ? *carry_in : T(0);
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            const bool chain = (c == G - 1) && (t + 1 < M);
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
                r_prev = has ? (prefix + lb.own) : lb.own;
                if (lane == 0) S::publish(rnd, k, tag, r_prev);
            }
            if (k >= STAGES) mbar_wait(&pre_free[s], (uint32_t)(((k - STAGES) / STAGES) & 1));
            if (lane == 0) {
                pre[s] = prefix;
                pre_has[s] = has ? 1 : 0;
                mbar_arrive(&pre_ready[s]);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ scanners
        const uint32_t wbase = (uint32_t)warp * WARP_BYTES + (uint32_t)lane * 16;  // row 0 of this lane
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const uint32_t parity = (uint32_t)((k / STAGES) & 1);
            const int64_t t = c + k * G;
            mbar_wait(&full[s], parity);
            if (p.delay_scan_ns > 0 && t % 3 == 2 && warp == (int)(t % SCAN_WARPS)) debug_sleep(p.delay_scan_ns);
            Regs<T, V> r;
            const uint32_t sbase = smem_u32(stages + s * TILE_BYTES) + wbase;
#pragma unroll
            for (int j = 0; j < V; ++j) r.q[j] = lds128(sbase + (uint32_t)j * 512u);
            // per row: lane-serial sum of the vector, inclusive warp scan of those
            T rex[V];  // exclusive prefix of this lane within row j (valid for lane > 0)
            T rtot[V];  // row totals
#pragma unroll
            for (int j = 0; j < V; ++j) {
                T v = r.e[j * PER];
#pragma unroll
                for (int e = 1; e < PER; ++e) v = v + r.e[j * PER + e];
                const T inc = warp_inclusive_scan(v, lane);
                rex[j] = __shfl_up_sync(0xffffffffu, inc, 1);
                rtot[j] = __shfl_sync(0xffffffffu, inc, 31);
            }
            // serial row carry (Alg. 2): running prefix of the rows before j
            T rowpre[V];
            T run = rtot[0];
            rowpre[0] = T(0);
#pragma unroll
            for (int j = 1; j < V; ++j) {
                rowpre[j] = run;
                run = run + rtot[j];
            }
            if (lane == 0) warp_tot[warp] = run;
            named_bar_sync(1, SCAN_THREADS);  // (A) stage fully read; warp totals visible
            if (tid == 0) {
                mbar_arrive(&empty[s]);
                if (k > 0) mbar_arrive(&pre_free[(k - 1) % STAGES]);
            }
            if (warp == 0) {
                const T wt = lane < SCAN_WARPS ? warp_tot[lane] : T(0);
                const T wi = warp_inclusive_scan(wt, lane);
                const T we = __shfl_up_sync(0xffffffffu, wi, 1);
                if (lane < SCAN_WARPS) warp_exc[lane] = we;
                if (t == M - 1 && p.total_out != nullptr) {
                    mbar_wait(&pre_ready[s], parity);
                    const T blk = __shfl_sync(0xffffffffu, wi, SCAN_WARPS - 1);
                    if (lane == 0) *static_cast<T *>(p.total_out) = pre_has[s] ? (pre[s] + blk) : blk;
                }
            }
            mbar_wait(&pre_ready[s], parity);
            named_bar_sync(1, SCAN_THREADS);  // (B)
            // carry into this lane's first element of each row:
            //   tile prefix (+) warps before (+) rows before (+) lanes before
            bool has0 = pre_has[s] != 0;
            T wcarry = pre[s];
            if (warp > 0) { wcarry = has0 ? (wcarry + warp_exc[warp]) : warp_exc[warp]; has0 = true; }
            T *yt = y + t * (int64_t)TILE_ELEMS;
            const bool partial = t >= full_tiles;
            const int64_t valid = p.n - t * (int64_t)TILE_ELEMS;
#pragma unroll
            for (int j = 0; j < V; ++j) {
                bool has = has0;
                T acc = wcarry;
                if (j > 0) { acc = has ? (acc + rowpre[j]) : rowpre[j]; has = true; }
                if (lane > 0) { acc = has ? (acc + rex[j]) : rex[j]; has = true; }
#pragma unroll
                for (int e = 0; e < PER; ++e) {
                    const T v = r.e[j * PER + e];
                    if (EXCL) {
                        r.e[j * PER + e] = (e == 0 && !has) ? T(0) : acc;
                        acc = (e == 0 && !has) ? v : (acc + v);
                    } else {
                        acc = (e == 0 && !has) ? v : (acc + v);
                        r.e[j * PER + e] = acc;
                    }
                }
                const int64_t vec = (int64_t)warp * (WARP_BYTES / 16) + j * 32 + lane;  // 16-byte vector index
                if (!partial || (vec + 1) * PER <= valid) {
                    stg128(reinterpret_cast<uint8_t *>(yt) + vec * 16, r.q[j]);
                } else if (vec * PER < valid) {
#pragma unroll
                    for (int e = 0; e < PER; ++e)
                        if (vec * PER + e < valid) yt[vec * PER + e] = r.e[j * PER + e];
                }
            }
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
constexpr size_t scan_ws2_smem_bytes() {
    return scan_ws_smem_bytes<T, SCAN_WARPS, TILE_BYTES, STAGES>();
}

}  // namespace lscan
