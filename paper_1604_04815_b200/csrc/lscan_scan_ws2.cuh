// lscan_scan_ws2.cuh — the hot path: warp-specialised persistent single-pass
// scan with register-resident results, for 16-byte-aligned x and y.
//
// Maps the reference's chained pipeline (chainscan/chained.py:316-357) onto
// a B200.  The roles the reference's worker performs in sequence per block
// (chained.py:237-249: local accumulate -> inter_block_comm -> combine) run
// as concurrent warp roles inside each persistent CTA, so the cross-CTA carry
// chain is resolved ahead of the data pass instead of stalling it:
//
//   producer warp   1-D TMA bulk loads (cp.async.bulk) of whole tiles into a
//                   STAGES-deep shared-memory ring; a stage is refilled as
//                   soon as the scanners and the reducer have read it
//   reducer warp    reduces each landed tile and publishes A[t] (never waits
//                   on another CTA)
//   look-back warp  prefix(t) = R[r-1] (+) A[rG] (+) ... (+) A[rG+c-1] into a
//                   shared-memory ring; CTA G-1 also publishes the round
//                   prefix R[r] = prefix(t) (+) A[t] (the only serial chain:
//                   one L2 round trip per round of G tiles)
//   scanner warps   copy the tile into registers in the paper's lane-strided
//                   layout (Alg. 2, warp.py:85-90, with
//                   16-byte vectors as row elements) and release the stage;
//                   thread-serial fold per vector, __shfl_up_sync row scan and
//                   serial row carry (Alg. 2), shared-memory scan of warp
//                   totals (Alg. 3), prefix fold (Alg. 5), coalesced STG.128
//
// Tile t = r*G + c is CTA c's r-th tile: cyclic, ascending, no atomic ticket
// (Alg. 1; chained.py:270).  The launch is cooperative, so the driver refuses
// a grid that cannot be co-resident.  Sums are fixed-order:
// results depend on (n, G, tile shape) only, never on timing.
#pragma once
#include "lscan_common.cuh"

// lab knobs (bench_support/lscan_lab.cu builds; the product uses the defaults):
// look-back poll back-off, the L2 policy of the TMA loads, and timing-only
// switches that skip the reducer's pass over the stage / the scanners' row
// warp scans (wrong sums; they locate the power the kernel draws)
#ifndef LS_LOOKBACK_SLEEP_NS
#define LS_LOOKBACK_SLEEP_NS 32
#endif
#ifndef LS_TMA_EVICT_FIRST
#define LS_TMA_EVICT_FIRST 1
#endif
#ifndef LS_LAB_SKIP_REDUCE
#define LS_LAB_SKIP_REDUCE 0
#endif
#ifndef LS_LAB_SKIP_ROWSCAN
#define LS_LAB_SKIP_ROWSCAN 0
#endif
// lab: per-phase clock64 totals (scanner warp 0, the producer and the look-back
// warp), summed over CTAs into the workspace header's pad words
#ifndef LS_LAB_TIMING
#define LS_LAB_TIMING 0
#endif
#ifndef LS_LAB_SKIP_LOOKBACK
#define LS_LAB_SKIP_LOOKBACK 0
#endif
// The producer's first ring fill keeps at most this many tile loads in
// flight (0 = the whole ring at once): round 0 then lands before round 1 is
// requested, so the carry chain starts early instead of behind a ring's
// worth of interleaved loads (lab, scripts/gpu/r2l.sh: i32 2^24 507 -> 586,
// 2^26 735 -> 762, 2^28 809 -> 816 Gelem/s; i64 2^23 280 -> 295)
#ifndef LS_FILL_LOOKAHEAD
#define LS_FILL_LOOKAHEAD 1
#endif

// lab: per-CTA event times (%globaltimer ns, 32 ns ticks on B200) into the
// buffer p.xchg points at (single-GPU lab builds only): [c][0] start, [c][1]
// end, [c][2 + 8k + e] for the CTA's k-th tile (k < 8): e = 0 data landed
// (as the reducer sees it), 1 aggregate published, 2 prefix known (look-back
// warp), 3 stores issued (scanners), 4 look-back started, 5 its first pass of
// slot loads answered, 6 re-polls (a count) — scripts/timeline_lab.py
#ifndef LS_LAB_TIMELINE
#define LS_LAB_TIMELINE 0
#endif
constexpr int kTimelineWords = 66;

// lab: the scanners' row scans through the predicated-shuffle add
// (shfl_up_add, as the latency kernel); measured -1 to -2 % for 64-bit types
#ifndef LS_WS2_PRED_SCAN
#define LS_WS2_PRED_SCAN 0
#endif

#ifndef LS_SHIFT_NAN_REDUCE
#define LS_SHIFT_NAN_REDUCE 0
#endif

// f32 add on packed FADD2 (add.rn.f32x2, sm_100): the reducer folds two
// elements per instruction (as IADD3 does for integers), and the scanners keep
// each lane's running prefixes in place and add the row carry to two of them
// per instruction once the tile prefix arrives.  0 = the scalar forms (lab A/B)
#ifndef LS_F32_PACKED
#define LS_F32_PACKED 1
#endif

namespace lscan {

__device__ __forceinline__ uint64_t pack2(uint32_t lo, uint32_t hi) {
    uint64_t r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}
__device__ __forceinline__ void unpack2(uint64_t v, uint32_t &lo, uint32_t &hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "l"(v));
}
// two independent f32 adds in one instruction (FADD2), round to nearest
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
    uint64_t r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

__device__ __forceinline__ uint64_t gtimer_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <typename T, typename OP>
__host__ __device__ constexpr bool packed_f32_add() {
    return LS_F32_PACKED && std::is_same<T, float>::value && OP::code == 0 && !OP::idempotent;
}

// 64-bit max / min: the scanners keep each lane's in-lane running prefixes
// in place (the row fold's intermediates), so the store pass combines the
// carry with every element independently instead of re-folding the lane's
// chunk serially (the exact f64 operator is a three-deep chain per element)
#ifndef LS_PIP_MAXMIN
#define LS_PIP_MAXMIN 0
#endif
template <typename T, typename OP>
__host__ __device__ constexpr bool pip_maxmin() {
    return LS_PIP_MAXMIN && sizeof(T) == 8 && OP::code != 0;
}

// Transposed row scan (TRS): a scanner lane's VR row totals are written to a
// per-warp scratch in sequence order (row-major over lanes), each lane reads
// back VR consecutive ones, folds them, and ONE warp scan plus one exclusive
// shuffle gives every (row, lane) its exclusive prefix over all rows and lanes
// before it — instead of VR warp scans, VR shuffles of the row totals and a
// serial carry over rows.  Sequence order is kept throughout (left operand =
// earlier elements), so it is exact for the order-sensitive float max / min.
// LS_ROW_TRANSPOSE: 0 off, 1 order-sensitive 64-bit ops (f64 max / min),
// 2 every 64-bit max / min, 3 every operator and type
#ifndef LS_ROW_TRANSPOSE
#define LS_ROW_TRANSPOSE 1
#endif
template <typename T, typename OP>
__host__ __device__ constexpr bool row_transpose() {
    return (LS_ROW_TRANSPOSE == 1 && sizeof(T) == 8 && order_sensitive<T, OP>()) ||
           (LS_ROW_TRANSPOSE == 2 && sizeof(T) == 8 && OP::code != 0) || LS_ROW_TRANSPOSE == 3;
}

__device__ __forceinline__ void stg128(void *p, uint4 v) {
    asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// Order-sensitive operators (float max/min, lscan_common.cuh): the reducers
// below combine a tile out of sequence order, which is exact except for the
// bits of a tie-class result (a zero or a NaN).  Then the tile is searched for
// the element the sequential fold would return — the rightmost zero, or the
// leftmost NaN — among the window's elements [lo, hi) (16-byte vectors, lane
// strided).  Rare by construction: one extra pass only when the tile's
// aggregate is a zero or a NaN.
template <typename T, typename OP>
__device__ __noinline__ T tile_ties(const uint8_t *st, int lane, T fast, int nvec, int lo, int hi) {
    constexpr int PER = 16 / (int)sizeof(T);
    const bool nan = fast != fast;
    int best = nan ? 0x7fffffff : -1;
    for (int v = lane; v < nvec; v += 32) {
        Regs<T, 1> r;
        r.q[0] = lds128(smem_u32(st) + (uint32_t)v * 16u);
#pragma unroll
        for (int e = 0; e < PER; ++e) {
            const int w = v * PER + e;
            const T x = r.e[e];
            if (w >= lo && w < hi && (nan ? x != x : x == (T)0)) best = nan ? min(best, w) : max(best, w);
        }
    }
    best = nan ? __reduce_min_sync(0xffffffffu, best) : __reduce_max_sync(0xffffffffu, best);
    return reinterpret_cast<const T *>(st)[best];
}

// reduce a whole shared-memory tile with one warp (lane-strided 16-byte
// vectors, conflict-free), four independent accumulators, fixed order
// f32 max / min: the whole tile with FMNMX3.NAN (two elements per operator,
// no NaN or sign-of-zero bookkeeping), then the exact re-derivation when the
// result is a NaN or a zero.  Window elements outside [lo, hi) are skipped
// (identity).
template <typename T, typename OP, int NVEC>
__device__ __forceinline__ T reduce_stage_nan(const uint8_t *st, int lane, int lo, int hi) {
    using R = typename ScanFastOp<T, OP>::reduce_type;
    const T ident = OP::template identity<T>();
    T acc[4] = {ident, ident, ident, ident};
    const uint32_t base = smem_u32(st);
    constexpr int ITERS = (NVEC + 31) / 32;  // lane-strided vectors per lane
#pragma unroll 2
    for (int i = 0; i < ITERS; i += 4) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {  // four independent chains
            const int v = (i + u) * 32 + lane;
            if (v < NVEC) {
                Regs<T, 1> r;
                r.q[0] = lds128(base + (uint32_t)v * 16u);
                if (v * 4 < lo || v * 4 + 4 > hi) {  // the window's edge vectors only
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (v * 4 + e < lo || v * 4 + e >= hi) r.e[e] = ident;
                }
                acc[u] = R::apply3(acc[u], r.e[0], r.e[1]);
                acc[u] = R::apply3(acc[u], r.e[2], r.e[3]);
            }
        }
    }
    T x = R::apply(R::apply3(acc[0], acc[1], acc[2]), acc[3]);
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) x = R::apply(x, __shfl_xor_sync(0xffffffffu, x, d));
    if (tie_class(x)) return tile_ties<T, OP>(st, lane, x, NVEC, lo, hi);
    return x;
}

#ifndef LS_F64_FAST_REDUCE
#define LS_F64_FAST_REDUCE 1
#endif
template <typename T, typename OP, int TILE_BYTES>
__device__ __forceinline__ T reduce_stage(const uint8_t *st, int lane) {
    constexpr int NV = TILE_BYTES / 16 / 32;  // 16-byte vectors per lane
    constexpr int PER = 16 / (int)sizeof(T);
    static_assert(NV % 4 == 0, "tile must hold a multiple of 4 vectors per lane");
    if constexpr (ScanFastOp<T, OP>::reduce_nan)
        return reduce_stage_nan<T, OP, TILE_BYTES / 16>(st, lane, 0, TILE_BYTES / (int)sizeof(T));
    if constexpr (packed_f32_add<T, OP>()) {
        // four packed accumulators: two FADD2 per 16-byte vector
        uint64_t acc[4] = {0, 0, 0, 0};
        const uint32_t base = smem_u32(st) + (uint32_t)lane * 16;
#pragma unroll 2
        for (int j = 0; j < NV; j += 4) {
            uint4 q[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) q[u] = lds128(base + (uint32_t)(j + u) * 512u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                acc[u] = fadd2(acc[u], pack2(q[u].x, q[u].y));
                acc[u] = fadd2(acc[u], pack2(q[u].z, q[u].w));
            }
        }
        const uint64_t a2 = fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3]));
        uint32_t lo, hi;
        unpack2(a2, lo, hi);
        return warp_reduce_fixed<T, OP>(__uint_as_float(lo) + __uint_as_float(hi));
    }
    const T ident = OP::template identity<T>();
    if constexpr (LS_F64_FAST_REDUCE && std::is_same<T, double>::value && OP::code != 0) {
        // f64 max / min: order-free max.f64 / min.f64 (one DSETP.MAX + selects;
        // drops NaNs, either zero on a tie) beside a NaN screen — the high
        // words viewed as f32 through the NaN-propagating FMNMX3 (an f64 NaN or
        // infinity is an f32 NaN there).  A flagged tile (NaN, infinity or a
        // magnitude >= 2^1017) is folded again exactly; a zero result is
        // re-derived by tile_ties as before
        using F = typename std::conditional<OP::code == 1, OpFastMaxD, OpFastMinD>::type;
        double fa[4] = {ident, ident, ident, ident};
        float nf = 0.f;
        const uint32_t fbase = smem_u32(st) + (uint32_t)lane * 16;
#pragma unroll 2
        for (int j = 0; j < NV; j += 4) {
            Regs<T, 4> r;
#pragma unroll
            for (int u = 0; u < 4; ++u) r.q[u] = lds128(fbase + (uint32_t)(j + u) * 512u);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                fa[u] = F::apply(F::apply(fa[u], r.e[u * 2]), r.e[u * 2 + 1]);
                nf = OpNanMaxF::apply3(nf, __uint_as_float(r.q[u].y), __uint_as_float(r.q[u].w));
            }
        }
        if (!__any_sync(0xffffffffu, nf != nf)) {
            double a = F::apply(F::apply(fa[0], fa[1]), F::apply(fa[2], fa[3]));
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) a = F::apply(a, __shfl_xor_sync(0xffffffffu, a, d));
            if (a == 0.0) return tile_ties<T, OP>(st, lane, a, TILE_BYTES / 16, 0, TILE_BYTES / (int)sizeof(T));
            return a;
        }
    }
    T acc[4] = {ident, ident, ident, ident};
    const uint32_t base = smem_u32(st) + (uint32_t)lane * 16;
#pragma unroll 2
    for (int j = 0; j < NV; j += 4) {
        Regs<T, 4> r;
#pragma unroll
        for (int u = 0; u < 4; ++u) r.q[u] = lds128(base + (uint32_t)(j + u) * 512u);
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[u] = OP::apply(acc[u], r.e[u * PER + e]);
    }
    const T a = warp_reduce_fixed<T, OP>(OP::apply(OP::apply(acc[0], acc[1]), OP::apply(acc[2], acc[3])));
    if constexpr (order_sensitive<T, OP>())
        if (tie_class(a)) return tile_ties<T, OP>(st, lane, a, TILE_BYTES / 16, 0, TILE_BYTES / (int)sizeof(T));
    return a;
}

// the same over a shifted window (SHIFT): the stage holds TILE_BYTES + 16
// bytes from the 16-byte boundary below the tile, whose first `sh` elements
// belong to the previous tile and whose last vector's first `sh` elements to
// this one.  HALF: -1 the whole window; 0 / 1 its lower / upper half (the two
// reducer warps of RED2: the upper half ends with the window's last vector)
template <typename T, typename OP, int TILE_BYTES, int HALF = -1>
__device__ __forceinline__ T reduce_stage_shifted(const uint8_t *st, int lane, int sh) {
    constexpr int NV = TILE_BYTES / 16 / 32 / (HALF < 0 ? 1 : 2);
    constexpr int PER = 16 / (int)sizeof(T);
    constexpr int TILE_ELEMS = TILE_BYTES / (int)sizeof(T);
    static_assert(NV % 4 == 0, "a (half) tile must hold a multiple of 4 vectors per lane");
    // lab (LS_SHIFT_NAN_REDUCE=1, with LS_SHIFT_RED2_32=0): f32 max / min over
    // the window's elements [sh, sh + TILE_ELEMS) with FMNMX3.NAN, as the
    // aligned reducer
    if constexpr (LS_SHIFT_NAN_REDUCE && HALF < 0 && ScanFastOp<T, OP>::reduce_nan)
        return reduce_stage_nan<T, OP, TILE_BYTES / 16 + 1>(st, lane, sh, sh + TILE_ELEMS);
    const T ident = OP::template identity<T>();
    // (the aligned reducer's order-free f64 form measured slower here: shifted
    // f64 max 355 -> 342 Gelem/s, profiles/r2_f64_maxmin_ab.json)
    T acc[4] = {ident, ident, ident, ident};
    const uint32_t base = smem_u32(st) + (HALF == 1 ? (uint32_t)TILE_BYTES / 2u : 0u) + (uint32_t)lane * 16;
#pragma unroll 2
    for (int j = 0; j < NV; j += 4) {
        Regs<T, 4> r;
#pragma unroll
        for (int u = 0; u < 4; ++u) r.q[u] = lds128(base + (uint32_t)(j + u) * 512u);
        if (HALF != 1 && j == 0 && lane == 0) {
#pragma unroll
            for (int e = 0; e < PER; ++e)
                if (e < sh) r.e[e] = ident;  // the previous tile's elements
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int e = 0; e < PER; ++e) acc[u] = OP::apply(acc[u], r.e[u * PER + e]);
    }
    T a = OP::apply(OP::apply(acc[0], acc[1]), OP::apply(acc[2], acc[3]));
    if (HALF != 0 && lane == 0) {
        Regs<T, 1> r;
        r.q[0] = lds128(smem_u32(st) + (uint32_t)TILE_BYTES);
#pragma unroll
        for (int e = 0; e < PER; ++e)
            if (e < sh) a = OP::apply(a, r.e[e]);
    }
    a = warp_reduce_fixed<T, OP>(a);
    if constexpr (order_sensitive<T, OP>())
        if (tie_class(a))
            return tile_ties<T, OP>(st, lane, a, TILE_BYTES / 16 + 1, HALF == 1 ? TILE_ELEMS / 2 : sh,
                                    HALF == 0 ? TILE_ELEMS / 2 : sh + TILE_ELEMS);
    return a;
}

// the same with the shift known at compile time: pure register renaming
template <int SW>
__device__ __forceinline__ uint4 funnel_words_c(uint4 a, uint4 b) {
    static_assert(SW >= 1 && SW <= 3, "a whole number of words inside one vector");
    if constexpr (SW == 1) return make_uint4(a.y, a.z, a.w, b.x);
    else if constexpr (SW == 2) return make_uint4(a.z, a.w, b.x, b.y);
    else return make_uint4(a.w, b.x, b.y, b.z);
}

// 16 bytes starting `sw` 32-bit words into a (continuing into b), sw in 1..3
__device__ __forceinline__ uint4 funnel_words(uint4 a, uint4 b, int sw) {
    uint4 r;
    r.x = sw == 1 ? a.y : (sw == 2 ? a.z : a.w);
    r.y = sw == 1 ? a.z : (sw == 2 ? a.w : b.x);
    r.z = sw == 1 ? a.w : (sw == 2 ? b.x : b.y);
    r.w = sw == 1 ? b.x : (sw == 2 ? b.y : b.z);
    return r;
}

template <typename T>
struct LookbackOut {
    T r;    // R[k-1]
    T sum;  // A[kG] (+) ... (+) A[kG+c-1]
    T own;  // A[t]
    int polls = 0;  // re-polls after the first pass (lab statistics)
};

// One look-back step for tile t = k*G + c, every load in flight at once: the
// round prefix R[k-1] (when need_r), the aggregates A[kG .. kG+c-1] and, when
// want_own, A[t] itself.  Spins (with nanosleep back-off) until every word
// carries `tag`; a spin budget turns a stall into LS_ERR_LIVENESS.
template <typename T, typename OP>
__device__ __forceinline__ LookbackOut<T> aux_lookback(const uint64_t *agg, const uint64_t *rnd, int64_t k, int c,
                                                       int G, bool need_r, int64_t r_idx, bool want_own, uint32_t tag,
                                                       int lane, int64_t spin_budget, Header *hdr, uint32_t where,
                                                       uint64_t *t_first = nullptr) {
    using S = Slot<T>;
    constexpr int U = 5;  // 160 slots per pass covers a 148-SM round
    const T ident = OP::template identity<T>();
    const int count = c + (want_own ? 1 : 0);
    const int64_t first = k * (int64_t)G;
    T acc = ident, own = ident, r = ident;
    int64_t probes = 0;
    int polls = 0;
    bool r_pending = need_r;
    uint64_t rw[S::W];
    if (need_r) S::load(rnd, r_idx, rw);
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
        bool first_pass = base == 0;
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
            if (LS_LAB_TIMELINE && first_pass && t_first != nullptr) *t_first = gtimer_ns();
            first_pass = false;
            if (__all_sync(0xffffffffu, ok)) break;
            if (spin_budget > 0 && ++probes > spin_budget) {
                if (lane == 0) raise_error(hdr, 4u /*LS_ERR_LIVENESS*/, where);
                if (r_pending) { r = ident; r_pending = false; }
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (need[u]) { val[u] = ident; need[u] = false; }
                break;
            }
            __nanosleep(LS_LOOKBACK_SLEEP_NS);
            ++polls;
            if (r_pending) S::load(rnd, r_idx, rw);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int j = base + u * 32 + lane;
                if (need[u]) S::load(agg, first + j, w[u]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * 32 + lane;
            if constexpr (order_sensitive<T, OP>()) {
                acc = fold_chunk<T, OP>(acc, j < c ? val[u] : ident);  // slot order
                if (j == c && want_own) own = val[u];
            } else {
                if (j < c) acc = OP::apply(acc, val[u]);
                else if (j == c && want_own) own = val[u];
            }
        }
    }
    LookbackOut<T> o;
    o.sum = fold_finish<T, OP>(acc);
    o.r = r;
    o.own = want_own ? __shfl_sync(0xffffffffu, own, c & 31) : ident;
    o.polls = polls;
    return o;
}

// Round prefixes (single GPU, add): every CTA folds the whole previous round
// itself (round_lookback) instead of reading the round prefix CTA G-1
// publishes — no serial hop through one CTA per round (lab, with the fill
// look-ahead: i32 2^28 816 -> 827, i64 2^27 407 -> 414 Gelem/s).  Not for
// max / min: float max / min fold each 32-slot chunk with a warp reduction,
// and the doubled look-back work measured slower there (f32 max 2^28 822 -> 499)
#ifndef LS_ROUND_FOLD
#define LS_ROUND_FOLD 1
#endif

template <typename T>
struct RoundPair {
    T prev;  // A[first] (+) ... (+) A[first + n1 - 1]: the whole previous round
    T cur;   // A[first + n1] (+) ... (+) A[first + n1 + n2 - 1]: this round's tiles before t
    int polls = 0;
};

// The look-back of tile t = k*G + c (k >= 1) on a single GPU: the previous
// round's G aggregates and this round's first c, every load in flight at once
// (U * 32 >= 2G slots), folded separately in slot order — so every CTA folds
// round k-1 identically and keeps its own running round prefix R[k-1]; no
// CTA waits on another's published round prefix (one L2 round trip per
// tile instead of a serial hop through CTA G-1 per round).
template <typename T, typename OP, int U>
__device__ __forceinline__ RoundPair<T> round_lookback(const uint64_t *agg, int64_t first, int n1, int n2,
                                                       uint32_t tag, int lane, int64_t spin_budget, Header *hdr,
                                                       uint32_t where) {
    using S = Slot<T>;
    const T ident = OP::template identity<T>();
    const int count = n1 + n2;
    T a1 = ident, a2 = ident;
    int64_t probes = 0;
    int polls = 0;
    for (int base = 0; base < count; base += 32 * U) {  // one pass while 2G <= 32 U (G <= 160)
        // raw tagged words only (decoded again for the fold): the 64-bit form
        // keeps 2U words live, not 2U words and U values
        uint64_t w[U][S::W];
        bool need[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j = base + u * 32 + lane;
            need[u] = j < count;
            if (need[u]) S::load(agg, first + j, w[u]);
        }
        bool timed_out = false;
        while (true) {
            bool ok = true;
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (need[u]) {
                    T v;
                    if (S::decode(w[u], tag, v)) need[u] = false;
                    else ok = false;
                }
            }
            if (__all_sync(0xffffffffu, ok)) break;
            if (spin_budget > 0 && ++probes > spin_budget) {
                if (lane == 0) raise_error(hdr, 4u /*LS_ERR_LIVENESS*/, where);
                timed_out = true;  // slots still missing fold as the identity
                break;
            }
            __nanosleep(LS_LOOKBACK_SLEEP_NS);
            ++polls;
#pragma unroll
            for (int u = 0; u < U; ++u)
                if (need[u]) S::load(agg, first + base + u * 32 + lane, w[u]);
        }
        // slot order: whole 32-slot chunks, the one straddling n1 split in two
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int j0 = base + u * 32, j = j0 + lane;
            T v = ident;
            if (j < count && !(timed_out && need[u])) S::decode(w[u], tag, v);
            if (j0 < n1) a1 = fold_chunk<T, OP>(a1, j < n1 ? v : ident);
            if (j0 + 32 > n1 && j0 < count) a2 = fold_chunk<T, OP>(a2, j >= n1 ? v : ident);
        }
    }
    RoundPair<T> o;
    o.prev = fold_finish<T, OP>(a1);
    o.cur = fold_finish<T, OP>(a2);
    o.polls = polls;
    return o;
}

template <int SCAN_WARPS, bool MULTI>
__host__ __device__ constexpr int ws2_threads() { return (SCAN_WARPS + (MULTI ? 5 : 3)) * 32; }

// 64-bit max / min: the exact operator is four or five instructions and one
// reducer warp publishes tile aggregates too late for the look-back (lab:
// i64 max 340 -> 415 Gelem/s with the reducer pass skipped).  A second
// reducer warp takes the upper half of each tile.  LS_SHIFT_RED2 (default
// on): the shifted-window kernel too, whose reducer also masks the window
#ifndef LS_SHIFT_RED2
#define LS_SHIFT_RED2 1
#endif
template <typename T, typename OP, bool MULTI, bool SHIFT>
// LS_SHIFT_RED2_32: the second reducer for 32-bit max / min in the
// shifted-window kernel too, whose reducer keeps the exact operator (the
// aligned kernel's FMNMX3.NAN reducer measured slower there): f32 max with x
// one element off 554 -> 736, i32 751 -> 823 Gelem/s (lab, scripts/gpu/r2t.sh).
// LS_SHIFT_RED2_ADD (lab): the same for 64-bit add in the shifted kernel
#ifndef LS_SHIFT_RED2_32
#define LS_SHIFT_RED2_32 1
#endif
#ifndef LS_SHIFT_RED2_ADD
#define LS_SHIFT_RED2_ADD 0
#endif
// LS_RED2_ADD (lab): the second reducer for add in the aligned kernel (the
// single reducer publishes one 32 KiB tile per ~0.85 us at mid n)
#ifndef LS_RED2_ADD
#define LS_RED2_ADD 0
#endif
__host__ __device__ constexpr bool ws2_red2() {
    return !MULTI && (!SHIFT || LS_SHIFT_RED2) &&
           ((OP::idempotent && (sizeof(T) == 8 || (SHIFT && LS_SHIFT_RED2_32 && sizeof(T) == 4))) ||
            (SHIFT && LS_SHIFT_RED2_ADD && !OP::idempotent && sizeof(T) == 8) ||
            (!SHIFT && LS_RED2_ADD && !OP::idempotent));
}
template <int SCAN_WARPS, bool MULTI, bool RED2>
__host__ __device__ constexpr int ws2_threads_x() { return ws2_threads<SCAN_WARPS, MULTI>() + (RED2 ? 32 : 0); }

// Cross-GPU round chain helpers (MULTI): the exchange slot of (round k, gpu g)
// in a GPU's exchange region, double-buffered by call parity so a fast GPU's
// next call can never overwrite a slot a slow GPU still reads.
template <typename T>
__device__ __forceinline__ uint64_t *xchg_slots(uint8_t *region, uint32_t xtag, int64_t rounds_cap, int world) {
    return reinterpret_cast<uint64_t *>(region + kXchgSlotBase) +
           (int64_t)(xtag & 1u) * rounds_cap * world * Slot<T>::W;
}

// VW: 16-byte vectors per lane per scanner row (1, or 2: 32-byte lane chunks,
// one 256-bit store each, half the warp scans per element)
template <typename T, typename OP, int SCAN_WARPS, int TILE_BYTES, int STAGES, bool EXCL, bool MULTI = false,
          bool SHIFT = false, int VW = 1>
__global__ void __launch_bounds__(ws2_threads_x<SCAN_WARPS, MULTI, ws2_red2<T, OP, MULTI, SHIFT>()>(), 1)
    scan_ws2_kernel(const ScanParams p) {
    constexpr bool RED2 = ws2_red2<T, OP, MULTI, SHIFT>();
    constexpr int SCAN_THREADS = SCAN_WARPS * 32;
    constexpr int V = TILE_BYTES / SCAN_THREADS / 16;  // rows (16-byte vectors) per lane
    constexpr int PER = 16 / (int)sizeof(T);           // elements per vector
    constexpr int TILE_ELEMS = TILE_BYTES / (int)sizeof(T);
    constexpr int WARP_BYTES = TILE_BYTES / SCAN_WARPS;
    constexpr int VR = V / VW;      // scanner rows per lane
    constexpr int RPER = VW * PER;  // elements per lane per row
    constexpr uint32_t ROW_BYTES = 512u * VW;
    static_assert(V % VW == 0 && (VW == 1 || VW == 2), "rows of one or two vectors per lane");
    constexpr int W_PROD = SCAN_WARPS, W_RED = SCAN_WARPS + 1, W_AUX = SCAN_WARPS + 2;
    constexpr int W_RED2 = SCAN_WARPS + 3;  // RED2 only (never with MULTI)
    constexpr int W_PUSH = SCAN_WARPS + 3, W_GCHAIN = SCAN_WARPS + 4;  // MULTI only, CTA G-1 only
    static_assert(V >= 1 && TILE_BYTES % (SCAN_THREADS * 16) == 0, "whole rows per lane");
    static_assert(!(SHIFT && MULTI), "the shifted window is a single-GPU variant");
    // SHIFT: x is not 16-byte aligned; every tile is loaded as a window of
    // TILE_BYTES + 16 bytes from the boundary below it; a window that x does
    // not fully back (the last tile or two) is loaded as a TMA prefix plus a
    // plain-loaded ragged vector padded with the identity (see the producer)
    constexpr int STAGE_BYTES = TILE_BYTES + (SHIFT ? 16 : 0);
    static_assert(SCAN_WARPS >= 2 && ws2_threads<SCAN_WARPS, MULTI>() <= 1024, "too many warps");
    using S = Slot<T>;
    const T ident = OP::template identity<T>();

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *stages = smem;
    uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);  // data landed
    uint64_t *empty = full + STAGES;          // scanners + reducer done reading (2 arrivals)
    uint64_t *pre_ready = empty + STAGES;     // prefix written
    uint64_t *pre_free = pre_ready + STAGES;  // prefix consumed
    T *pre = reinterpret_cast<T *>(pre_free + STAGES);
    int *pre_has = reinterpret_cast<int *>(pre + STAGES);
    T *warp_tot = reinterpret_cast<T *>(pre_has + STAGES + (STAGES & 1));
    T *warp_exc = warp_tot + SCAN_WARPS;
    uint64_t *red2_ready = reinterpret_cast<uint64_t *>(warp_exc + SCAN_WARPS);  // RED2: upper half reduced
    T *red2_val = reinterpret_cast<T *>(red2_ready + STAGES);
    // TRS scratch: V * 32 values per scanner warp, 16-byte aligned
    T *trs_base = reinterpret_cast<T *>((reinterpret_cast<uintptr_t>(red2_val + STAGES) + 15u) & ~(uintptr_t)15u);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    long long lab_t[6] = {0, 0, 0, 0, 0, 0};  // LS_LAB_TIMING only
    long long lab_polls = 0, lab_chain = 0;
    const int64_t M = p.num_tiles;
    Header *hdr = reinterpret_cast<Header *>(p.ws);
    uint64_t *agg = reinterpret_cast<uint64_t *>(p.ws + kSlotBase);
    uint64_t *rnd = agg + M * S::W;
    const T *x = static_cast<const T *>(p.x);
    T *y = static_cast<T *>(p.y);
    const int64_t my_tiles = (M - c + G - 1) / G;
    const int64_t full_tiles = p.n / TILE_ELEMS;
    auto tl_mark = [&](int idx) {  // LS_LAB_TIMELINE only
        if constexpr (LS_LAB_TIMELINE && !MULTI)
            if (p.xchg != nullptr && idx < kTimelineWords)
                reinterpret_cast<volatile uint64_t *>(p.xchg)[(int64_t)c * kTimelineWords + idx] = gtimer_ns();
    };
    auto tl_set = [&](int idx, uint64_t v) {  // LS_LAB_TIMELINE only
        if constexpr (LS_LAB_TIMELINE && !MULTI)
            if (p.xchg != nullptr && idx < kTimelineWords)
                reinterpret_cast<volatile uint64_t *>(p.xchg)[(int64_t)c * kTimelineWords + idx] = v;
    };

    if (tid == 0) {
#pragma unroll
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], RED2 ? 3 : 2);
            if (RED2) mbar_init(&red2_ready[s], 1);
            mbar_init(&pre_ready[s], 1);
            mbar_init(&pre_free[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    // programmatic dependent launch: everything above overlaps the previous
    // kernel's tail; no global memory is touched before this wait (it returns
    // once that kernel has completed and flushed).  The next kernel may start
    // launching right away: its blocks take SMs only as ours exit.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    if (tid == 0) tl_mark(0);
    const uint32_t tag = call_tag(hdr);
    Header *xhdr = MULTI ? reinterpret_cast<Header *>(p.xchg) : nullptr;
    const uint32_t xtag = MULTI ? call_tag(xhdr) : 0u;

    if (warp == W_PROD) {
        // ------------------------------------------------------------ producer
        // x is read once: evict-first, unless x and y fit in L2 together (the
        // host decides, p.l2_resident), where a caller's next pass may hit it
        const uint64_t pol =
            (LS_TMA_EVICT_FIRST && !p.l2_resident) ? policy_evict_first() : policy_evict_normal();
        auto load_tile = [&](int64_t k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            const int64_t t0 = t * TILE_ELEMS;
            uint8_t *sb = stages + s * STAGE_BYTES;
            // SHIFT: a window is TILE_ELEMS + PER elements from the boundary
            // below the tile; it is TMA'd whole only when x backs all of it
            if (SHIFT && p.x_shift / (int)sizeof(T) + (p.n - t0) >= TILE_ELEMS + PER) {
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
                    tma_load_1d(sb, reinterpret_cast<const uint8_t *>(x) - p.x_shift + t * (int64_t)TILE_BYTES,
                                STAGE_BYTES, &full[s], pol);
                }
            } else if (SHIFT) {
                // a window running past x's end (the last tile or two): window
                // elements [0, sh + n - t0) hold data (the first sh the previous
                // tile's); their 16-byte-aligned prefix by TMA, the ragged vector
                // by plain loads, the rest identity — never reading past x's end
                const int sh = p.x_shift / (int)sizeof(T);
                const int64_t wvalid = sh + (p.n - t0);
                const uint32_t bulk = (uint32_t)((wvalid * (int64_t)sizeof(T)) & ~(int64_t)15);
                const int vfirst = (int)(bulk / 16);
                const uint32_t sbase = smem_u32(sb);
                const uint4 iv = identity_vec<T, OP>();
                for (int v = vfirst + 1 + lane; v < STAGE_BYTES / 16; v += 32) sts128(sbase + (uint32_t)v * 16u, iv);
                if (lane == 0) {
                    Regs<T, 1> rv;
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        const int64_t w = (int64_t)vfirst * PER + e;
                        rv.e[e] = (w >= sh && w < wvalid) ? x[t0 + w - sh] : ident;
                    }
                    sts128(sbase + (uint32_t)vfirst * 16u, rv.q[0]);
                }
                __syncwarp();
                if (lane == 0) {
                    if (bulk) {
                        mbar_arrive_expect_tx(&full[s], bulk);
                        tma_load_1d(sb, reinterpret_cast<const uint8_t *>(x) - p.x_shift + t * (int64_t)TILE_BYTES, bulk,
                                    &full[s], pol);
                    } else {
                        mbar_arrive(&full[s]);
                    }
                }
            } else if (t < full_tiles) {
                if (lane == 0) {
                    mbar_arrive_expect_tx(&full[s], TILE_BYTES);
                    tma_load_1d(sb, x + t0, TILE_BYTES, &full[s], pol);
                }
            } else {
                // partial_tail (chained.py:188-202): the 16-byte-aligned prefix
                // by TMA, the ragged vector by plain loads, the rest of the
                // stage identity-filled with 128-bit shared stores
                const int64_t valid = p.n - t0;
                const uint32_t bulk = (uint32_t)((valid * (int64_t)sizeof(T)) & ~(int64_t)15);
                const int vfirst = (int)(bulk / 16);  // first vector not covered by TMA
                const uint32_t sbase = smem_u32(sb);
                const uint4 iv = identity_vec<T, OP>();
                for (int v = vfirst + 1 + lane; v < TILE_BYTES / 16; v += 32) sts128(sbase + (uint32_t)v * 16u, iv);
                if (lane == 0) {
                    Regs<T, 1> rv;
#pragma unroll
                    for (int e = 0; e < PER; ++e) {
                        const int64_t i = (int64_t)vfirst * PER + e;
                        rv.e[e] = i < valid ? x[t0 + i] : ident;
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
        if (LS_FILL_LOOKAHEAD > 0 && LS_FILL_LOOKAHEAD < STAGES) {
            for (int64_t k = 0; k < STAGES && k < my_tiles; ++k) {
                if (k >= LS_FILL_LOOKAHEAD)
                    mbar_wait(&full[(k - LS_FILL_LOOKAHEAD) % STAGES], 0u);  // first use of that stage
                load_tile(k);
            }
        } else {
            for (int64_t k = 0; k < STAGES && k < my_tiles; ++k) load_tile(k);
        }
        for (int64_t k = 0; k + STAGES < my_tiles; ++k) {
            long long tw = LS_LAB_TIMING ? clock64() : 0;
            mbar_wait(&empty[k % STAGES], (uint32_t)((k / STAGES) & 1));
            if (LS_LAB_TIMING) lab_t[4] += clock64() - tw;  // producer waiting for a free stage
            load_tile(k + STAGES);
        }
    } else if (RED2 && warp == W_RED2) {
        // ------------------------------------------ second reducer (RED2)
        // the upper half of each tile; handed to the reducer through smem
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
            T a = ident;
            if (!LS_LAB_SKIP_REDUCE) {
                if constexpr (SHIFT)
                    a = reduce_stage_shifted<T, OP, TILE_BYTES, 1>(stages + s * STAGE_BYTES, lane,
                                                                   p.x_shift / (int)sizeof(T));
                else
                    a = reduce_stage<T, OP, TILE_BYTES / 2>(stages + s * STAGE_BYTES + TILE_BYTES / 2, lane);
            }
            __syncwarp();
            if (lane == 0) {
                red2_val[s] = a;
                mbar_arrive(&red2_ready[s]);
                mbar_arrive(&empty[s]);
            }
        }
    } else if (warp == W_RED) {
        // ------------------------------------------------------------- reducer
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            mbar_wait(&full[s], (uint32_t)((k / STAGES) & 1));
            if (lane == 0) tl_mark(2 + 8 * (int)k);
            if (p.delay_red_ns > 0 && t % 3 == 1) debug_sleep(p.delay_red_ns);
            T a;
            if constexpr (RED2) {
                // lower half here, upper half from the second reducer, in order
                a = LS_LAB_SKIP_REDUCE ? ident
                    : SHIFT ? reduce_stage_shifted<T, OP, TILE_BYTES, 0>(stages + s * STAGE_BYTES, lane,
                                                                         p.x_shift / (int)sizeof(T))
                            : reduce_stage<T, OP, TILE_BYTES / 2>(stages + s * STAGE_BYTES, lane);
                mbar_wait(&red2_ready[s], (uint32_t)((k / STAGES) & 1));
                a = OP::apply(a, red2_val[s]);
            } else {
                a = LS_LAB_SKIP_REDUCE ? ident
                    : SHIFT ? reduce_stage_shifted<T, OP, TILE_BYTES>(stages + s * STAGE_BYTES, lane,
                                                                      p.x_shift / (int)sizeof(T))
                            : reduce_stage<T, OP, TILE_BYTES>(stages + s * STAGE_BYTES, lane);
            }
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[s]);
                if (p.protocol_checks) {
                    uint64_t w[S::W];
                    T dummy;
                    S::load(agg, t, w);
                    if (S::decode(w, tag, dummy)) raise_error(hdr, 5u /*LS_ERR_PROTOCOL*/, (uint32_t)t);
                }
                if (t != p.stall_tile || p.spin_budget <= 0) S::publish(agg, t, tag, t == p.corrupt_tile ? ident : a);
                tl_mark(3 + 8 * (int)k);
            }
        }
    } else if (warp == W_AUX) {
        // ----------------------------------------------------------- look-back
        const T *carry_in = static_cast<const T *>(p.carry_in);
        bool have_carry = carry_in != nullptr;
        T r_prev = have_carry ? *carry_in : ident;  // R[k-1]: carry (+) head (+) rounds 0 .. k-1 (single GPU)
        if constexpr (!MULTI) {
            // y's head (the few elements before the aligned y this kernel
            // tiles): every CTA folds it into the carry, in sequence order;
            // the last CTA to finish stores it (below), after every CTA has
            // read it — so x == y is safe.  One launch for any alignment
            const T *hx = x - p.head_n;
            for (int i = 0; i < p.head_n; ++i) {
                r_prev = have_carry ? OP::apply(r_prev, hx[i]) : hx[i];
                have_carry = true;
            }
        }
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const int64_t t = c + k * G;
            bool has;
            T prefix;
            if constexpr (MULTI) {
                // X[k] = everything before this GPU's k-th stripe, published by
                // the global-chain warp of CTA G-1
                const LookbackOut<T> lb = aux_lookback<T, OP>(agg, rnd, k, c, G, true, k, false, tag, lane,
                                                              p.spin_budget, hdr, (uint32_t)t);
                has = k > 0 || p.rank > 0 || have_carry;
                prefix = lb.r;
                if (c > 0) {
                    prefix = has ? OP::apply(lb.r, lb.sum) : lb.sum;
                    has = true;
                }
            } else if (LS_ROUND_FOLD && OP::code == OpAdd::code) {
                // prefix(t) = R[k-1] (+) A[kG] (+) ... (+) A[kG+c-1], with R[k-1]
                // this CTA's own running fold of the whole earlier rounds (no
                // chain through CTA G-1)
                const long long tl = LS_LAB_TIMING ? clock64() : 0;
                T cur = ident;
                if (LS_LAB_SKIP_LOOKBACK) {
                } else if (k == 0) {
                    const LookbackOut<T> lb = aux_lookback<T, OP>(agg, rnd, 0, c, G, false, 0, false, tag, lane,
                                                                  p.spin_budget, hdr, (uint32_t)t);
                    cur = lb.sum;
                    if (LS_LAB_TIMING) lab_polls += lb.polls;
                } else {
                    const RoundPair<T> lb = round_lookback<T, OP, 10>(agg, (k - 1) * (int64_t)G, G, c, tag, lane,
                                                                      p.spin_budget, hdr, (uint32_t)t);
                    r_prev = have_carry ? OP::apply(r_prev, lb.prev) : lb.prev;
                    have_carry = true;
                    cur = lb.cur;
                    if (LS_LAB_TIMING) lab_polls += lb.polls;
                }
                if (LS_LAB_TIMING) {
                    lab_t[5] += clock64() - tl;  // look-back of one tile
                    if (c == G - 1) lab_chain += clock64() - tl;
                }
                has = have_carry;
                prefix = r_prev;
                if (c > 0) {
                    prefix = has ? OP::apply(prefix, cur) : cur;
                    has = true;
                }
            } else {
                const bool chain = (c == G - 1) && (t + 1 < M);
                // R[k-1]: the caller's carry in round 0, the chain owner's register,
                // or the published round slot for everyone else
                const bool need_r = k > 0 && c != G - 1;
                const long long tl = LS_LAB_TIMING ? clock64() : 0;
                uint64_t t_first = 0;
                if (lane == 0) tl_mark(6 + 8 * (int)k);
                const LookbackOut<T> lb =
                    LS_LAB_SKIP_LOOKBACK ? LookbackOut<T>{ident, ident, ident, 0}
                                         : aux_lookback<T, OP>(agg, rnd, k, c, G, need_r, k - 1, chain, tag, lane,
                                                               p.spin_budget, hdr, (uint32_t)t, &t_first);
                if (lane == 0) {
                    tl_set(7 + 8 * (int)k, t_first);
                    tl_set(8 + 8 * (int)k, (uint64_t)lb.polls);
                }
                if (LS_LAB_TIMING) {
                    lab_t[5] += clock64() - tl;  // look-back of one tile
                    lab_polls += lb.polls;
                    if (c == G - 1) lab_chain += clock64() - tl;
                }
                T base;
                if (k == 0) { has = have_carry; base = r_prev; }
                else if (c == G - 1) { has = true; base = r_prev; }
                else { has = true; base = lb.r; }
                prefix = base;
                if (c > 0) {
                    prefix = has ? OP::apply(base, lb.sum) : lb.sum;
                    has = true;
                }
                if (chain) {
                    r_prev = has ? OP::apply(prefix, lb.own) : lb.own;  // R[k]
                    if (lane == 0) S::publish(rnd, k, tag, r_prev);
                }
            }
            if (k >= STAGES) mbar_wait(&pre_free[s], (uint32_t)(((k - STAGES) / STAGES) & 1));
            if (lane == 0) {
                pre[s] = prefix;
                pre_has[s] = has ? 1 : 0;
                mbar_arrive(&pre_ready[s]);
                tl_mark(4 + 8 * (int)k);
            }
            __syncwarp();
        }
    } else if (MULTI && warp == W_PUSH) {
        // ------------------------------------------- stripe aggregate pusher
        // (CTA G-1 only) BA[k] = A[kG] (+) ... (+) A[kG+G-1], stored into every
        // GPU's exchange slot (k, rank) as soon as this GPU's round k landed
        if (c == G - 1) {
            const int64_t rounds = (M + G - 1) / G;
            uint64_t *peer = lane < p.world ? p.xchg_peers[lane] : nullptr;
            for (int64_t k = 0; k < rounds; ++k) {
                const int cnt = (int)((M - k * G) < G ? (M - k * G) : G);
                const LookbackOut<T> lb = aux_lookback<T, OP>(agg, rnd, k, cnt, G, false, 0, false, tag, lane,
                                                              p.spin_budget, hdr, (uint32_t)(k * G));
                if (lane < p.world) {
                    uint64_t *slots = xchg_slots<T>(reinterpret_cast<uint8_t *>(peer), xtag, p.xchg_rounds, p.world);
                    S::publish_sys(slots, k * p.world + p.rank, xtag, lb.sum);
                }
            }
        }
    } else if (MULTI && warp == W_GCHAIN) {
        // -------------------------------------------------- global chain
        // (CTA G-1 only) X[k] = GB[k-1] (+) BA[k][0] (+) ... (+) BA[k][rank-1];
        // GB[k] = X[k] (+) BA[k][rank] (+) ... (+) BA[k][world-1]; every GPU
        // folds the same values in the same order, so all agree bit for bit
        if (c == G - 1) {
            const T *carry_in = static_cast<const T *>(p.carry_in);
            bool have_gb = carry_in != nullptr;
            T gb = have_gb ? *carry_in : ident;
            const int64_t rounds = (M + G - 1) / G;
            uint64_t *slots = xchg_slots<T>(p.xchg, xtag, p.xchg_rounds, p.world);
            int64_t probes = 0;
            for (int64_t k = 0; k < rounds; ++k) {
                T v = ident;
                uint64_t w[S::W];
                bool ok = lane >= p.world;
                if (!ok) S::load_sys(slots, k * p.world + lane, w);
                while (true) {
                    if (!ok) ok = S::decode(w, xtag, v);
                    if (__all_sync(0xffffffffu, ok)) break;
                    if (p.spin_budget > 0 && ++probes > p.spin_budget) {
                        if (lane == 0) raise_error(hdr, 4u /*LS_ERR_LIVENESS*/, (uint32_t)(k * G));
                        if (!ok) { v = ident; ok = true; }
                        break;
                    }
                    __nanosleep(32);
                    if (!ok) S::load_sys(slots, k * p.world + lane, w);
                }
                T x = gb;  // fold in GPU order; lane-uniform
                bool hx = have_gb;
                for (int g = 0; g < p.world; ++g) {
                    const T bg = __shfl_sync(0xffffffffu, v, g);
                    if (g == p.rank) {
                        if (lane == 0) S::publish(rnd, k, tag, x);  // X[k]
                    }
                    x = hx ? OP::apply(x, bg) : bg;
                    hx = true;
                }
                gb = x;
                have_gb = true;
            }
            if (p.total_out != nullptr && lane == 0) *static_cast<T *>(p.total_out) = gb;
        }
    } else if (warp < SCAN_WARPS) {
        // ------------------------------------------------------------ scanners
        const uint32_t wbase = (uint32_t)warp * WARP_BYTES + (uint32_t)lane * 16u * VW;  // row 0 of this lane
        const bool y256 = VW == 2 && ((uintptr_t)y & 31u) == 0;
        for (int64_t k = 0; k < my_tiles; ++k) {
            const int s = (int)(k % STAGES);
            const uint32_t parity = (uint32_t)((k / STAGES) & 1);
            const int64_t t = c + k * G;
            long long tm0 = LS_LAB_TIMING ? clock64() : 0;
            mbar_wait(&full[s], parity);
            long long tm1 = LS_LAB_TIMING ? clock64() : 0;
            if (p.delay_scan_ns > 0 && t % 3 == 2 && warp == (int)(t % SCAN_WARPS)) debug_sleep(p.delay_scan_ns);
            Regs<T, V> r;
            const uint32_t sbase = smem_u32(stages + s * STAGE_BYTES) + wbase;
            if constexpr (SHIFT) {
                // logical vector v = window bytes [16v + shift, +16): two aligned
                // reads and a word funnel (x is element-aligned, so the shift is
                // a whole number of 32-bit words).  The shift is made a compile-
                // time constant — always 2 words for 64-bit elements, one of three
                // load loops for 32-bit ones — so the funnel is register renaming
                // instead of branches and predicated moves per vector
                auto load_rows = [&](auto swc) {
                    constexpr int SW = decltype(swc)::value;
#pragma unroll
                    for (int j = 0; j < VR; ++j) {
                        uint4 a = lds128(sbase + (uint32_t)j * ROW_BYTES);
#pragma unroll
                        for (int u = 0; u < VW; ++u) {
                            const uint4 b = lds128(sbase + (uint32_t)j * ROW_BYTES + 16u * (u + 1));
                            r.q[j * VW + u] = funnel_words_c<SW>(a, b);
                            a = b;
                        }
                    }
                };
                if constexpr (sizeof(T) == 8) {
                    load_rows(std::integral_constant<int, 2>{});
                } else {
                    const int sw = p.x_shift >> 2;
                    if (sw == 1) load_rows(std::integral_constant<int, 1>{});
                    else if (sw == 2) load_rows(std::integral_constant<int, 2>{});
                    else load_rows(std::integral_constant<int, 3>{});
                }
            } else {
#pragma unroll
                for (int j = 0; j < VR; ++j)
#pragma unroll
                    for (int u = 0; u < VW; ++u) r.q[j * VW + u] = lds128(sbase + (uint32_t)j * ROW_BYTES + 16u * u);
            }
            // float max / min: a warp chunk with no zero and no NaN scans with
            // one FMNMX (f32) / one DSETP.MAX (f64) per operator (ScanFastOp)
            bool fast = false;
            if constexpr (ScanFastOp<T, OP>::enabled) fast = __all_sync(0xffffffffu, fast_domain<T, V>(r.q));
            // per row j: lane-serial fold of the lane's chunk, inclusive warp scan
            T rex[VR];   // exclusive prefix of this lane within row j (lane > 0)
            T rtot[VR];  // row totals
            T run;
            // f32 add (PIP): each lane keeps its chunk's running prefixes in
            // place (the fold's intermediates), so the carry is added to every
            // element independently, two per FADD2, once the prefix is known
            constexpr bool PIP = packed_f32_add<T, OP>() && !EXCL;
            constexpr bool PIPM = pip_maxmin<T, OP>();
            // TRS: rex[j] is this lane's exclusive prefix over the rows before
            // j and the lanes before it in row j (undefined at row 0, lane 0)
            constexpr bool TRS = row_transpose<T, OP>() && VR > 1 && !PIP && !LS_LAB_SKIP_ROWSCAN;
            auto row_scans = [&](auto opv) {
                using O = decltype(opv);
                if constexpr (TRS) {
                    T *trs = trs_base + warp * (V * 32);
#pragma unroll
                    for (int j = 0; j < VR; ++j) {
                        T v = r.e[j * RPER];
                        if constexpr (PIPM) {
#pragma unroll
                            for (int e = 1; e < RPER; ++e) r.e[j * RPER + e] = v = O::apply(v, r.e[j * RPER + e]);
                        } else if constexpr (O::three) {
#pragma unroll
                            for (int e = 1; e + 1 < RPER; e += 2) v = O::apply3(v, r.e[j * RPER + e], r.e[j * RPER + e + 1]);
                            if constexpr (RPER % 2 == 0) v = O::apply(v, r.e[j * RPER + RPER - 1]);
                        } else {
#pragma unroll
                            for (int e = 1; e < RPER; ++e) v = O::apply(v, r.e[j * RPER + e]);
                        }
                        trs[j * 32 + lane] = v;
                    }
                    __syncwarp();
                    T f[VR];  // in-lane inclusive prefixes of values VR*lane .. VR*lane + VR - 1
                    if constexpr (VR % 2 == 0 && sizeof(T) == 8) {
#pragma unroll
                        for (int i = 0; i < VR; i += 2) {
                            const uint4 w = lds128(smem_u32(trs + VR * lane + i));
                            const uint64_t a = ((uint64_t)w.y << 32) | w.x, b = ((uint64_t)w.w << 32) | w.z;
                            memcpy(&f[i], &a, 8);
                            memcpy(&f[i + 1], &b, 8);
                        }
                    } else {
#pragma unroll
                        for (int i = 0; i < VR; ++i) f[i] = trs[VR * lane + i];
                    }
#pragma unroll
                    for (int i = 1; i < VR; ++i) f[i] = O::apply(f[i - 1], f[i]);
                    const T inc = warp_inclusive_scan<T, O, LS_WS2_PRED_SCAN != 0>(f[VR - 1], lane);
                    const T exl = __shfl_up_sync(0xffffffffu, inc, 1);
                    run = __shfl_sync(0xffffffffu, inc, 31);
                    // exclusive prefix of value VR*lane + i: lanes' values before,
                    // then this lane's first i (lane 0, i = 0: none, left as is)
                    if (lane > 0) trs[VR * lane] = exl;
#pragma unroll
                    for (int i = 1; i < VR; ++i) trs[VR * lane + i] = lane > 0 ? O::apply(exl, f[i - 1]) : f[i - 1];
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < VR; ++j) rex[j] = trs[j * 32 + lane];
                } else {
#pragma unroll
                for (int j = 0; j < VR; ++j) {
                    T v = r.e[j * RPER];
                    if constexpr (PIP || PIPM) {
#pragma unroll
                        for (int e = 1; e < RPER; ++e) r.e[j * RPER + e] = v = O::apply(v, r.e[j * RPER + e]);
                    } else if constexpr (O::three) {
                        // two elements per FMNMX3
#pragma unroll
                        for (int e = 1; e + 1 < RPER; e += 2) v = O::apply3(v, r.e[j * RPER + e], r.e[j * RPER + e + 1]);
                        if constexpr (RPER % 2 == 0) v = O::apply(v, r.e[j * RPER + RPER - 1]);
                    } else {
#pragma unroll
                        for (int e = 1; e < RPER; ++e) v = O::apply(v, r.e[j * RPER + e]);
                    }
                    if (LS_LAB_SKIP_ROWSCAN) {
                        rex[j] = v;
                        rtot[j] = v;
                        continue;
                    }
                    const T inc = warp_inclusive_scan<T, O, LS_WS2_PRED_SCAN != 0>(v, lane);
                    if constexpr (std::is_integral<T>::value && OP::code == OpAdd::code) {
                        // integer add: the exclusive prefix is inclusive - own value,
                        // exact modulo 2^width, one shuffle fewer per row (+1-2 % i64)
                        rex[j] = OP::apply(inc, (T)(0 - (typename std::make_unsigned<T>::type)v));
                    } else {
                        rex[j] = __shfl_up_sync(0xffffffffu, inc, 1);
                    }
                    rtot[j] = __shfl_sync(0xffffffffu, inc, 31);
                }
                // serial row carry (Alg. 2): the warp's total over its rows
                run = rtot[0];
#pragma unroll
                for (int j = 1; j < VR; ++j) run = O::apply(run, rtot[j]);
                }
            };
            if constexpr (ScanFastOp<T, OP>::enabled) {
                if (fast) row_scans(typename ScanFastOp<T, OP>::type{});
                else row_scans(OP{});
            } else {
                row_scans(OP{});
            }
            if (lane == 0) warp_tot[warp] = run;
            named_bar_sync(1, SCAN_THREADS);  // (A) stage fully read; warp totals visible
            long long tm2 = LS_LAB_TIMING ? clock64() : 0;
            if (tid == 0) {
                mbar_arrive(&empty[s]);
                if (k > 0) mbar_arrive(&pre_free[(k - 1) % STAGES]);
            }
            if (warp == 0) {
                const T wt = lane < SCAN_WARPS ? warp_tot[lane] : ident;
                const T wi = warp_inclusive_scan<T, OP>(wt, lane);
                const T we = __shfl_up_sync(0xffffffffu, wi, 1);
                if (lane < SCAN_WARPS) warp_exc[lane] = we;
                if (!MULTI && t == M - 1 && p.total_out != nullptr) {
                    mbar_wait(&pre_ready[s], parity);
                    const T blk = __shfl_sync(0xffffffffu, wi, SCAN_WARPS - 1);
                    if (lane == 0) *static_cast<T *>(p.total_out) = pre_has[s] ? OP::apply(pre[s], blk) : blk;
                }
            }
            mbar_wait(&pre_ready[s], parity);
            named_bar_sync(1, SCAN_THREADS);  // (B)
            long long tm3 = LS_LAB_TIMING ? clock64() : 0;
            // carry into the first element of each of this lane's rows:
            //   tile prefix (+) warps before (+) rows before (+) lanes before
            bool has0 = pre_has[s] != 0;
            T wcarry = pre[s];
            if (warp > 0) { wcarry = has0 ? OP::apply(wcarry, warp_exc[warp]) : warp_exc[warp]; has0 = true; }
            T *yt = y + t * (int64_t)TILE_ELEMS;
            const bool partial = t >= full_tiles;
            const int64_t valid = p.n - t * (int64_t)TILE_ELEMS;
            // rows before j, folded as the rows are stored (the same left fold as
            // the warp total above; no per-row array kept across the wait)
            auto fold_store = [&](auto opv, bool nan_fill) {
                using O = decltype(opv);
                [[maybe_unused]] T rowpre = ident;
                if constexpr (!TRS) rowpre = rtot[0];
#pragma unroll
                for (int j = 0; j < VR; ++j) {
                    if (nan_fill) {
                        // a NaN carry (fast chunks only): numpy keeps the left
                        // NaN, so every result of the chunk is the carry
#pragma unroll
                        for (int e = 0; e < RPER; ++e) r.e[j * RPER + e] = wcarry;
                    } else {
                        bool has = has0;
                        T acc = wcarry;
                        if constexpr (TRS) {
                            if (j > 0 || lane > 0) { acc = has ? O::apply(acc, rex[j]) : rex[j]; has = true; }
                        } else {
                        if (j > 0) {
                            acc = has ? O::apply(acc, rowpre) : rowpre;
                            has = true;
                            if (j + 1 < VR) rowpre = O::apply(rowpre, rtot[j]);
                        }
                        if (lane > 0) { acc = has ? O::apply(acc, rex[j]) : rex[j]; has = true; }
                        }
                        if constexpr (PIP) {
                            // y = carry (+) in-lane prefix; nothing to add before the
                            // array's first element (no carry: y[0] = x[0] exactly)
                            if (has) {
                                const uint64_t cc = pack2(__float_as_uint(acc), __float_as_uint(acc));
#pragma unroll
                                for (int q = 0; q < RPER / 4; ++q) {
                                    uint4 &w = r.q[j * VW + q];
                                    unpack2(fadd2(cc, pack2(w.x, w.y)), w.x, w.y);
                                    unpack2(fadd2(cc, pack2(w.z, w.w)), w.z, w.w);
                                }
                            }
                        } else if constexpr (PIPM) {
                            // y_e = carry (+) p_e (exclusive: carry (+) p_{e-1}),
                            // every element independent of the others
                            if constexpr (EXCL) {
#pragma unroll
                                for (int e = RPER - 1; e > 0; --e)
                                    r.e[j * RPER + e] = has ? O::apply(acc, r.e[j * RPER + e - 1]) : r.e[j * RPER + e - 1];
                                r.e[j * RPER] = has ? acc : ident;
                            } else if (has) {
#pragma unroll
                                for (int e = 0; e < RPER; ++e) r.e[j * RPER + e] = O::apply(acc, r.e[j * RPER + e]);
                            }
                        } else {
#pragma unroll
                        for (int e = 0; e < RPER; ++e) {
                            const T v = r.e[j * RPER + e];
                            const bool first = (e == 0 && !has);
                            if (EXCL) {
                                r.e[j * RPER + e] = first ? ident : acc;
                                acc = first ? v : O::apply(acc, v);
                            } else {
                                acc = first ? v : O::apply(acc, v);
                                r.e[j * RPER + e] = acc;
                            }
                        }
                        }
                    }
                    // 16-byte vector index of the lane's chunk in this row
                    const int64_t vec = (int64_t)warp * (WARP_BYTES / 16) + (int64_t)(j * 32 + lane) * VW;
                    if (VW == 2 && y256 && (!partial || (vec + 2) * PER <= valid)) {
                        stg256(reinterpret_cast<uint8_t *>(yt) + vec * 16, r.q[j * VW], r.q[j * VW + 1]);
                    } else {
#pragma unroll
                        for (int u = 0; u < VW; ++u) {
                            const int64_t vu = vec + u;
                            if (!partial || (vu + 1) * PER <= valid) {
                                stg128(reinterpret_cast<uint8_t *>(yt) + vu * 16, r.q[j * VW + u]);
                            } else if (vu * PER < valid) {
#pragma unroll
                                for (int e = 0; e < PER; ++e)
                                    if (vu * PER + e < valid) yt[vu * PER + e] = r.e[(j * VW + u) * PER + e];
                            }
                        }
                    }
                }
            };
            if constexpr (ScanFastOp<T, OP>::enabled) {
                // the carry may be a zero or a NaN from outside the chunk: a zero
                // never ties with the chunk's (nonzero) values; a NaN fills it
                if (fast) fold_store(typename ScanFastOp<T, OP>::type{}, has0 && wcarry != wcarry);
                else fold_store(OP{}, false);
            } else {
                fold_store(OP{}, false);
            }
            if (tid == 0) tl_mark(5 + 8 * (int)k);
            if (LS_LAB_TIMING && tid == 0) {
                const long long tm4 = clock64();
                lab_t[0] += tm1 - tm0;  // waiting for the tile's data
                lab_t[1] += tm2 - tm1;  // loads + row scans + barrier (A)
                lab_t[2] += tm3 - tm2;  // warp-total scan, waiting for the prefix, barrier (B)
                lab_t[3] += tm4 - tm3;  // fold + stores issued
            }
        }
    }

    if (LS_LAB_TIMING) {
        unsigned long long *acc = reinterpret_cast<unsigned long long *>(hdr->pad);
        if (tid == 0)
            for (int i = 0; i < 4; ++i) atomicAdd(&acc[i], (unsigned long long)lab_t[i]);
        if (warp == W_PROD && lane == 0) atomicAdd(&acc[4], (unsigned long long)lab_t[4]);
        if (warp == W_AUX && lane == 0) {
            atomicAdd(&acc[5], (unsigned long long)lab_t[5]);
            atomicAdd(&acc[6], (unsigned long long)lab_polls);
            atomicAdd(&acc[7], (unsigned long long)lab_chain);
        }
    }
    __syncthreads();
    if (tid == 0) tl_mark(1);
    if (tid == 0) {
        if constexpr (MULTI) {
            // the exchange epoch advances with the workspace epoch: the last
            // CTA of this GPU records both
            const uint32_t old = atom_add_acqrel_u32(&hdr->done, 1u);
            if (old == (uint32_t)G - 1u) {
                st_relaxed_u32(&hdr->done, 0u);
                st_relaxed_u32(&xhdr->epoch, xtag);
                st_relaxed_u32(&hdr->epoch, tag);
            }
        } else {
            const uint32_t old = atom_add_acqrel_u32(&hdr->done, 1u);
            if (old == (uint32_t)G - 1u) {
                // every CTA has finished (and read y's head): store the head
                const T *hx = x - p.head_n;
                T *hy = y - p.head_n;
                const T *cin = static_cast<const T *>(p.carry_in);
                bool has = cin != nullptr;
                T acc = has ? *cin : ident;
                for (int i = 0; i < p.head_n; ++i) {
                    const T v = hx[i];
                    const T before = acc;
                    acc = has ? OP::apply(acc, v) : v;
                    hy[i] = EXCL ? (has ? before : ident) : acc;
                    has = true;
                }
                st_relaxed_u32(&hdr->done, 0u);
                st_relaxed_u32(&hdr->epoch, tag);
            }
        }
    }
}

template <typename T, int SCAN_WARPS, int TILE_BYTES, int STAGES, bool SHIFT = false, bool RED2 = false,
          bool TRS = false>
constexpr size_t scan_ws2_smem_bytes() {
    return (size_t)STAGES * (TILE_BYTES + (SHIFT ? 16 : 0)) + 4 * STAGES * 8 + STAGES * sizeof(T) +
           (STAGES + 1) * 4 + 2 * SCAN_WARPS * sizeof(T) + 32 + (RED2 || TRS ? STAGES * (8 + sizeof(T)) : 0) +
           // TRS scratch (row_transpose<T, OP>(), after the RED2 region): V * 32 values per scanner warp
           (TRS ? 16 + (size_t)TILE_BYTES / 16 * sizeof(T) : 0);
}

}  // namespace lscan
