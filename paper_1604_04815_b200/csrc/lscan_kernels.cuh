// lscan_kernels.cuh — the single-pass sum-scan for sm_100a.
//
// Maps the reference's chained pipeline (chainscan/chained.py:316-357) onto a
// B200:
//
//   reference (CPU re-enactment)              this kernel
//   ---------------------------------------   ---------------------------------------------
//   B persistent workers, block i owned by    grid = co-resident CTAs (cooperative launch),
//   worker i mod B (chained.py:264-287)       tile t owned by CTA t mod G, ascending
//   block_len L = K*W*warps (warp.py:42-82)   tile = TILE_BYTES of x (32 KiB), staged in
//                                             shared memory by 1-D TMA bulk copies, STAGES deep
//   local accumulate (chained.py:241-243,     thread-serial reduce of a register tile ->
//   warp.py:112-149)                          __shfl_up_sync warp scan -> smem scan of warp totals
//   inter_block_comm (chained.py:153-172)     round look-back over epoch-tagged 64-bit slots
//   CommSlots (chained.py:85-150)             in L2 (gpu-scope single-copy-atomic words)
//   combine(left, seg) (chained.py:248-249,   carry-seeded serial fold in registers, written
//   warp.py:152-169)                          back to smem, TMA bulk store to y
//   partial_tail (chained.py:188-202)         identity-filled generic load of the last tile
//
// Round look-back.  With G CTAs, tile t = r*G + c is CTA c's r-th tile
// ("round" r).  Every tile publishes its aggregate A[t] as soon as its local
// reduction is known; CTA G-1 additionally publishes the round prefix
// R[r] = (everything through tile r*G + G-1).  Tile t's exclusive prefix is
//     P(t) = R[r-1] (+) (A[rG] (+) ... (+) A[rG+c-1])
// summed by one warp in a fixed order.  This bounds every look-back to one
// round (at most G-1 aggregates read in parallel + one round slot), never
// spins on a tile of an earlier round except through R, and makes float
// results independent of timing: the association depends only on (n, G).
//
// Slots are written once per call and tagged with the call's epoch in the
// high half of each 64-bit word, so a reader either sees its epoch (value
// valid, same word) or keeps polling; no memset between calls.  64-bit
// element types use two such words (one per 32-bit half).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#include "lscan_ptx.cuh"

namespace lscan {

// ------------------------------------------------------------------------------
// element arithmetic: integers in unsigned registers (two's-complement wrap,
// operators.py:74-100), floats in IEEE add (no contraction involved)
template <typename T>
struct Elem;
template <>
struct Elem<uint32_t> {
    __device__ static uint32_t bits(uint32_t v) { return v; }
    __device__ static uint32_t from(uint32_t b) { return b; }
};
template <>
struct Elem<float> {
    __device__ static uint32_t bits(float v) { return __float_as_uint(v); }
    __device__ static float from(uint32_t b) { return __uint_as_float(b); }
};
template <>
struct Elem<uint64_t> {
    __device__ static uint64_t bits(uint64_t v) { return v; }
    __device__ static uint64_t from(uint64_t b) { return b; }
};
template <>
struct Elem<double> {
    __device__ static uint64_t bits(double v) { return (uint64_t)__double_as_longlong(v); }
    __device__ static double from(uint64_t b) { return __longlong_as_double((long long)b); }
};

// ------------------------------------------------------------------------------
// workspace layout (bytes):
//   [0, 128)                               Header
//   [128, 128 + kMaxGrid*8)                reduce partials (raw values, untagged)
//   [kSlotBase, kSlotBase + M*SW)          tile aggregate slots A[t]
//   [.., + M*SW)                           round prefix slots R[r]   (rounds <= M)
// SW = 8 (32-bit T) or 16 (64-bit T).  Partials live apart from the tagged
// slots so a raw value can never be mistaken for an epoch tag.
struct Header {
    uint32_t epoch;      // last completed call's tag (0 after init)
    uint32_t done;       // CTAs finished in the current call
    uint32_t error;      // first ls_status error code raised on the device
    uint32_t error_tile; // tile (or slot) index of that error
    uint32_t pad[28];
};
static_assert(sizeof(Header) == 128, "header is one 128-byte line");

constexpr int kMaxGrid = 4096;
constexpr size_t kSlotBase = sizeof(uint32_t) * 32 + (size_t)kMaxGrid * 8;

struct ScanParams {
    const void *x;
    void *y;
    int64_t n;
    const void *carry_in;   // device scalar or nullptr
    void *total_out;        // device scalar or nullptr
    uint8_t *ws;
    int64_t num_tiles;      // M
    int64_t spin_budget;    // 0 = unlimited
    int64_t corrupt_tile;   // -1 = off
    int protocol_checks;
    int experiment;         // lab-only bits: 1 = skip the look-back (timing upper bound, wrong sums)
    int64_t delay_red_ns;   // debug: reducer sleeps this long on tiles t % 3 == 1 (timing perturbation)
    int64_t delay_scan_ns;  // debug: scanners sleep this long on tiles t % 3 == 2
    int64_t stall_tile;     // debug: this tile never publishes its aggregate (needs a spin budget)
};

__device__ __forceinline__ void debug_sleep(int64_t ns) {
    while (ns > 0) {
        const unsigned chunk = ns > 100000 ? 100000u : (unsigned)ns;
        __nanosleep(chunk);
        ns -= chunk;
    }
}

template <typename T>
struct Slot {
    static constexpr int W = sizeof(T) / 4;  // 64-bit words per slot
    __device__ static void publish(uint64_t *arr, int64_t idx, uint32_t tag, T v) {
        uint64_t *p = arr + idx * W;
        uint64_t b = (uint64_t)Elem<T>::bits(v);
        if constexpr (W == 1) {
            slot_st(p, ((uint64_t)tag << 32) | (b & 0xffffffffull));
        } else {
            slot_st(p, ((uint64_t)tag << 32) | (b & 0xffffffffull));
            slot_st(p + 1, ((uint64_t)tag << 32) | (b >> 32));
        }
    }
    // raw words -> (valid, value)
    __device__ static bool decode(const uint64_t (&w)[W], uint32_t tag, T &v) {
        if constexpr (W == 1) {
            v = Elem<T>::from((uint32_t)w[0]);
            return (uint32_t)(w[0] >> 32) == tag;
        } else {
            v = Elem<T>::from((w[0] & 0xffffffffull) | (w[1] << 32));
            return (uint32_t)(w[0] >> 32) == tag && (uint32_t)(w[1] >> 32) == tag;
        }
    }
    __device__ static void load(const uint64_t *arr, int64_t idx, uint64_t (&w)[W]) {
        const uint64_t *p = arr + idx * W;
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] = slot_ld(p + i);
    }
};

__device__ __forceinline__ void raise_error(Header *h, uint32_t code, uint32_t where) {
    if (atomicCAS(&h->error, 0u, code) == 0u) h->error_tile = where;
}

// ------------------------------------------------------------------------------
// barrel rotation of a thread's 16-byte vectors (bank-conflict-free LDS/STS
// of a thread-contiguous tile): a'[i] = a[(i + r) mod V]
template <int V>
__device__ __forceinline__ void rotate_left(uint4 (&a)[V], int r) {
#pragma unroll
    for (int b = 1; b < V; b <<= 1) {
        const bool take = (r & b) != 0;
        uint4 t[V];
#pragma unroll
        for (int i = 0; i < V; ++i) t[i] = a[(i + b) % V];
#pragma unroll
        for (int i = 0; i < V; ++i) {
            a[i].x = take ? t[i].x : a[i].x;
            a[i].y = take ? t[i].y : a[i].y;
            a[i].z = take ? t[i].z : a[i].z;
            a[i].w = take ? t[i].w : a[i].w;
        }
    }
}

// rotation that spreads the 8 threads of one LDS.128 phase over all 32 banks
template <int V>
__device__ __forceinline__ int vec_rot(int tid) {
    if constexpr (V >= 8) return tid & 7;
    else if constexpr (V == 1) return 0;
    else return (tid / (8 / V)) & (V - 1);
}

template <typename T, int V>
union Regs {
    uint4 q[V];
    T e[V * 16 / sizeof(T)];
};

template <typename T, int V>
__device__ __forceinline__ void load_tile_regs(const uint8_t *stage, int tid, Regs<T, V> &r) {
    const int rot = vec_rot<V>(tid);
    const uint32_t base = smem_u32(stage) + (uint32_t)tid * (V * 16);
#pragma unroll
    for (int u = 0; u < V; ++u) r.q[u] = lds128(base + (uint32_t)(((u + rot) & (V - 1)) * 16));
    // r.q[u] holds vector (u + rot) mod V; un-rotate so r.q[j] holds vector j
    rotate_left<V>(r.q, (V - rot) & (V - 1));
}

template <typename T, int V>
__device__ __forceinline__ void store_tile_regs(uint8_t *stage, int tid, Regs<T, V> &r) {
    const int rot = vec_rot<V>(tid);
    const uint32_t base = smem_u32(stage) + (uint32_t)tid * (V * 16);
    rotate_left<V>(r.q, rot);  // r.q[u] now holds vector (u + rot) mod V
#pragma unroll
    for (int u = 0; u < V; ++u) sts128(base + (uint32_t)(((u + rot) & (V - 1)) * 16), r.q[u]);
}

template <typename T>
__device__ __forceinline__ T warp_inclusive_scan(T v, int lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v = o + v;  // lower-index operand first (operators.py:13-15)
    }
    return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum_fixed(T v) {
    // fixed xor-butterfly: every lane ends with bit-identical sums because
    // each level adds a commutative pair
#pragma unroll
    for (int d = 16; d >= 1; d >>= 1) v = v + __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// ------------------------------------------------------------------------------
// Round look-back, executed by one full warp.  Returns (has_prefix, prefix)
// for tile t = r*G + c.  Spins until every needed slot carries `tag`.
template <typename T>
__device__ __forceinline__ bool round_lookback(const uint64_t *agg, const uint64_t *rnd, int64_t r, int c,
                                               int G, uint32_t tag, const T *carry_in, int lane,
                                               int64_t spin_budget, Header *hdr, T &prefix) {
    using S = Slot<T>;
    constexpr int U = 4;  // slots in flight per lane per pass
    T acc = T(0);
    int64_t probes = 0;
    bool dead = false;
    const int64_t base_t = r * (int64_t)G;
    for (int base = 0; base < c; base += 32 * U) {
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
                    if (need[u]) { val[u] = T(0); need[u] = false; }
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
            if (j < c) acc = acc + val[u];  // lane-serial, ascending j
        }
        if (dead) break;
    }
    const T asum = warp_sum_fixed(acc);
    // previous round's prefix (or the caller's carry for round 0)
    bool has = false;
    T rp = T(0);
    if (r > 0) {
        uint64_t w[S::W];
        S::load(rnd, r - 1, w);
        while (!S::decode(w, tag, rp)) {
            if (spin_budget > 0 && ++probes > spin_budget) {
                if (lane == 0) raise_error(hdr, 4u, (uint32_t)(base_t + c));
                rp = T(0);
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
        prefix = has ? (rp + asum) : asum;
        return true;
    }
    prefix = rp;
    return has;
}

// ------------------------------------------------------------------------------
// The persistent single-pass scan kernel.
//   THREADS     CTA size
//   TILE_BYTES  bytes of x per tile (THREADS * V * 16)
//   STAGES      depth of the TMA load ring
//   EXCL        exclusive (true) or inclusive (false) scan
//   USE_TMA     bulk copies for full tiles (x, y 16-byte aligned); false =
//               generic element loads/stores everywhere (any alignment)
template <typename T, int THREADS, int TILE_BYTES, int STAGES, bool EXCL, bool USE_TMA>
__global__ void __launch_bounds__(THREADS, 1) scan_kernel(const ScanParams p) {
    constexpr int NWARPS = THREADS / 32;
    constexpr int V = TILE_BYTES / THREADS / 16;       // 16-byte vectors per thread
    constexpr int ITEMS = V * 16 / (int)sizeof(T);     // elements per thread
    constexpr int TILE_ELEMS = TILE_BYTES / (int)sizeof(T);
    constexpr int PRODUCER = THREADS - 32;             // lane 0 of the last warp
    static_assert(V >= 1 && (V & (V - 1)) == 0, "vectors per thread must be a power of two");
    static_assert(NWARPS <= 32 && NWARPS >= 2, "2..32 warps");
    static_assert(STAGES >= 2, "need at least double buffering");
    using S = Slot<T>;

    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t *stages = smem;
    uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + STAGES * TILE_BYTES);
    T *warp_tot = reinterpret_cast<T *>(full_bar + STAGES);  // [NWARPS]
    T *warp_exc = warp_tot + NWARPS;                         // [NWARPS]
    T *tile_pre = warp_exc + NWARPS;                         // [1]
    int *tile_has = reinterpret_cast<int *>(tile_pre + 1);   // [1]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = gridDim.x, c = blockIdx.x;
    const int64_t M = p.num_tiles;
    Header *hdr = reinterpret_cast<Header *>(p.ws);
    uint64_t *agg = reinterpret_cast<uint64_t *>(p.ws + kSlotBase);
    uint64_t *rnd = agg + M * S::W;
    const T *x = static_cast<const T *>(p.x);
    T *y = static_cast<T *>(p.y);
    const T *carry_in = static_cast<const T *>(p.carry_in);

    const uint32_t prev_epoch = ld_relaxed_u32(&hdr->epoch);
    const uint32_t tag = (prev_epoch + 1u) == 0u ? 1u : prev_epoch + 1u;

    const int64_t my_tiles = (M - c + G - 1) / G;
    const int64_t full_tiles = p.n / TILE_ELEMS;  // tiles with TILE_ELEMS valid elements
    uint64_t pol = 0;

    if (tid == PRODUCER) {
        pol = policy_evict_first();
#pragma unroll
        for (int s = 0; s < STAGES; ++s) mbar_init(&full_bar[s], 1);
        fence_mbar_init();
        if (USE_TMA) {
            for (int64_t k = 0; k < STAGES && k < my_tiles; ++k) {
                const int64_t t = c + k * G;
                if (t < full_tiles) {
                    mbar_arrive_expect_tx(&full_bar[k], TILE_BYTES);
                    tma_load_1d(stages + k * TILE_BYTES, x + t * TILE_ELEMS, TILE_BYTES, &full_bar[k], pol);
                }
            }
        }
    }
    __syncthreads();

    for (int64_t k = 0; k < my_tiles; ++k) {
        const int s = (int)(k % STAGES);
        const uint32_t parity = (uint32_t)((k / STAGES) & 1);
        const int64_t t = c + k * G;
        const bool generic = !USE_TMA || t >= full_tiles;
        uint8_t *st = stages + s * TILE_BYTES;
        const int64_t t0 = t * TILE_ELEMS;
        int64_t valid = p.n - t0;
        if (valid > TILE_ELEMS) valid = TILE_ELEMS;

        if (!generic) {
            mbar_wait(&full_bar[s], parity);
        } else {
            // partial_tail (chained.py:188-202): identity-padded tile
            T *sv = reinterpret_cast<T *>(st);
            for (int i = tid; i < TILE_ELEMS; i += THREADS) sv[i] = (i < valid) ? x[t0 + i] : T(0);
            __syncthreads();
        }

        Regs<T, V> r;
        load_tile_regs<T, V>(st, tid, r);

        // thread-serial reduction of the register tile
        T tsum = r.e[0];
#pragma unroll
        for (int i = 1; i < ITEMS; ++i) tsum = tsum + r.e[i];
        // warp scan of thread totals (Alg. 2 role), smem scan of warp totals (Alg. 3)
        const T winc = warp_inclusive_scan(tsum, lane);
        const T wexc = __shfl_up_sync(0xffffffffu, winc, 1);
        if (lane == 31) warp_tot[warp] = winc;
        __syncthreads();  // (A) warp totals visible; everyone is done reading stage `st`

        if (warp == 0) {
            const T wt = lane < NWARPS ? warp_tot[lane] : T(0);
            const T wi = warp_inclusive_scan(wt, lane);
            const T we = __shfl_up_sync(0xffffffffu, wi, 1);
            const T tile_agg = __shfl_sync(0xffffffffu, wi, NWARPS - 1);
            if (lane < NWARPS) warp_exc[lane] = we;
            // publish this tile's aggregate (Alg. 4 role, write-once slot)
            if (lane == 0) {
                if (p.protocol_checks) {
                    uint64_t w[S::W];
                    T dummy;
                    S::load(agg, t, w);
                    if (S::decode(w, tag, dummy)) raise_error(hdr, 5u /*LS_ERR_PROTOCOL*/, (uint32_t)t);
                }
                if (t != p.stall_tile || p.spin_budget <= 0) S::publish(agg, t, tag, t == p.corrupt_tile ? T(0) : tile_agg);
            }
            T prefix = T(0);
            const bool has = (p.experiment & 1)
                                 ? false
                                 : round_lookback<T>(agg, rnd, k, c, G, tag, carry_in, lane, p.spin_budget, hdr, prefix);
            const T incl = has ? (prefix + tile_agg) : tile_agg;
            if (lane == 0) {
                if (c == G - 1 && t + 1 < M) S::publish(rnd, k, tag, incl);
                if (t == M - 1 && p.total_out != nullptr) *static_cast<T *>(p.total_out) = incl;
                *tile_pre = prefix;
                *tile_has = has ? 1 : 0;
            }
        } else if (USE_TMA && tid == PRODUCER && k >= 1) {
            // refill the stage the previous tile used, once its TMA store has
            // finished reading shared memory (overlaps warp 0's look-back)
            bulk_wait_read<0>();
            const int64_t kn = k - 1 + STAGES;
            if (kn < my_tiles) {
                const int64_t tn = c + kn * G;
                if (tn < full_tiles) {
                    const int sn = (int)((k - 1) % STAGES);
                    mbar_arrive_expect_tx(&full_bar[sn], TILE_BYTES);
                    tma_load_1d(stages + sn * TILE_BYTES, x + tn * TILE_ELEMS, TILE_BYTES, &full_bar[sn], pol);
                }
            }
        }
        __syncthreads();  // (B) tile prefix + warp exclusive prefixes visible

        // carry-seeded serial fold (Alg. 5 role): acc starts at everything
        // before this thread's first element
        bool has = *tile_has != 0;
        T acc = *tile_pre;
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
        store_tile_regs<T, V>(st, tid, r);

        if (!generic) {
            fence_proxy_async_smem();
            __syncthreads();  // (C) tile results in smem
            if (tid == PRODUCER) {
                tma_store_1d(y + t0, st, TILE_BYTES, pol);
                bulk_commit();
            }
        } else {
            __syncthreads();
            const T *sv = reinterpret_cast<const T *>(st);
            for (int i = tid; i < valid; i += THREADS) y[t0 + i] = sv[i];
        }
    }

    if (tid == PRODUCER) bulk_wait_all();
    // epoch hand-over: the last CTA to finish records this call's tag
    if (tid == 0) {
        const uint32_t old = atom_add_acqrel_u32(&hdr->done, 1u);
        if (old == (uint32_t)G - 1u) {
            st_relaxed_u32(&hdr->done, 0u);
            st_relaxed_u32(&hdr->epoch, tag);
        }
    }
}

// ------------------------------------------------------------------------------
// Deterministic grid reduction (the per-shard total for the multi-GPU carry
// exchange).  Thread-serial over a fixed grid-stride partition, fixed warp and
// block trees, last CTA folds the per-CTA partials in index order.
template <typename T, int THREADS>
__global__ void __launch_bounds__(THREADS) reduce_kernel(const T *__restrict__ x, int64_t n, T *total_out,
                                                         uint8_t *ws) {
    constexpr int NWARPS = THREADS / 32;
    constexpr int PER_VEC = 16 / (int)sizeof(T);
    __shared__ T wsum[NWARPS];
    __shared__ bool last;
    Header *hdr = reinterpret_cast<Header *>(ws);
    T *partials = reinterpret_cast<T *>(ws + sizeof(Header));
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t gtid = (int64_t)blockIdx.x * THREADS + tid;
    const int64_t gstride = (int64_t)gridDim.x * THREADS;

    // head: elements before the first 16-byte boundary
    const int64_t mis = (int64_t)(((uintptr_t)x & 15u) / sizeof(T));
    int64_t head = mis ? (PER_VEC - mis) : 0;
    if (head > n) head = n;
    const int64_t nvec = (n - head) / PER_VEC;
    const int64_t tail0 = head + nvec * PER_VEC;
    T acc = T(0);
    if (gtid < head) acc = x[gtid];
    const uint4 *xv = reinterpret_cast<const uint4 *>(x + head);
    int64_t i = gtid;
    for (; i + 3 * gstride < nvec; i += 4 * gstride) {
        Regs<T, 4> q;
#pragma unroll
        for (int u = 0; u < 4; ++u) q.q[u] = __ldcs(xv + i + u * gstride);
#pragma unroll
        for (int j = 0; j < 4 * PER_VEC; ++j) acc = acc + q.e[j];
    }
    for (; i < nvec; i += gstride) {
        Regs<T, 1> q;
        q.q[0] = __ldcs(xv + i);
#pragma unroll
        for (int j = 0; j < PER_VEC; ++j) acc = acc + q.e[j];
    }
    if (gtid < n - tail0) acc = acc + x[tail0 + gtid];

    acc = warp_sum_fixed(acc);
    if (lane == 0) wsum[warp] = acc;
    __syncthreads();
    if (warp == 0) {
        T v = lane < NWARPS ? wsum[lane] : T(0);
        v = warp_sum_fixed(v);
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
        T v = T(0);
        for (int b = lane; b < (int)gridDim.x; b += 32) v = v + *((volatile T *)&partials[b]);
        v = warp_sum_fixed(v);
        if (lane == 0) {
            *total_out = v;
            st_relaxed_u32(&hdr->done, 0u);
        }
    }
}

// carry_out = totals[0] (+) ... (+) totals[rank-1]  (fixed left fold)
template <typename T>
__global__ void carry_kernel(const T *totals, int64_t rank, T *carry_out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        T acc = T(0);
        if (rank > 0) acc = totals[0];
        for (int64_t g = 1; g < rank; ++g) acc = acc + totals[g];
        *carry_out = acc;
    }
}

}  // namespace lscan
