// lscan_common.cuh — pieces shared by every scan kernel: element types and
// scan operators, the workspace layout, the epoch-tagged carry-chain slots,
// register-tile helpers and warp-level scans.
//
// Operators mirror chainscan/operators.py:111-127: add (identity 0; integers
// wrap modulo 2^width, operators.py:74-100), max (identity = lowest value,
// -inf for floats) and min (highest, +inf).  apply(a, b) takes the
// lower-index operand first (operators.py:13-15).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <type_traits>

#include "lscan_ptx.cuh"

namespace lscan {

// ------------------------------------------------------------------------------
// element bit casts (the slot protocol moves raw bits)
template <typename T>
struct Elem;
template <>
struct Elem<int32_t> {
    using Bits = uint32_t;
    __device__ static Bits bits(int32_t v) { return (uint32_t)v; }
    __device__ static int32_t from(Bits b) { return (int32_t)b; }
};
template <>
struct Elem<float> {
    using Bits = uint32_t;
    __device__ static Bits bits(float v) { return __float_as_uint(v); }
    __device__ static float from(Bits b) { return __uint_as_float(b); }
};
template <>
struct Elem<int64_t> {
    using Bits = uint64_t;
    __device__ static Bits bits(int64_t v) { return (uint64_t)v; }
    __device__ static int64_t from(Bits b) { return (int64_t)b; }
};
template <>
struct Elem<double> {
    using Bits = uint64_t;
    __device__ static Bits bits(double v) { return (uint64_t)__double_as_longlong(v); }
    __device__ static double from(Bits b) { return __longlong_as_double((long long)b); }
};

// ------------------------------------------------------------------------------
// scan operators (ls_op in include/lscan.h: 0 add, 1 max, 2 min)
struct OpAdd {
    static constexpr int code = 0;
    static constexpr bool idempotent = false;
    static constexpr bool three = false;  // no three-input form (apply3)
    template <typename T>
    __device__ __forceinline__ static T apply(T a, T b) {
        if constexpr (std::is_integral<T>::value) {
            using U = typename std::make_unsigned<T>::type;
            return (T)((U)a + (U)b);  // two's-complement wrap, no UB
        } else {
            return a + b;
        }
    }
    template <typename T>
    __device__ __forceinline__ static T identity() { return T(0); }
};

// numpy's float maximum / minimum (numpy 2.3, pinned by tests/test_ties_gpu.py):
//   maximum(a, b) = (a > b || isnan(a)) ? a : b      minimum: a < b
// equal operands give the RIGHT one (max(-0, +0) = +0, max(+0, -0) = -0) and a NaN
// on the left wins over one on the right.  As one predicate chain: FSETP.NAN,
// FSETP.GT.OR, FSEL (the C++ form compiles to a PLOP3 more).  FMNMX is not
// usable: it drops NaNs and orders -0 < +0.
template <typename T, bool GT>
__device__ __forceinline__ T float_keep_a(T a, T b) {
    T r;
    if constexpr (std::is_same<T, float>::value) {
        if constexpr (GT)
            asm("{\n .reg .pred p;\n setp.nan.f32 p, %1, %1;\n setp.gt.or.f32 p, %1, %2, p;\n"
                " selp.f32 %0, %1, %2, p;\n}" : "=f"(r) : "f"(a), "f"(b));
        else
            asm("{\n .reg .pred p;\n setp.nan.f32 p, %1, %1;\n setp.lt.or.f32 p, %1, %2, p;\n"
                " selp.f32 %0, %1, %2, p;\n}" : "=f"(r) : "f"(a), "f"(b));
    } else {
        if constexpr (GT)
            asm("{\n .reg .pred p;\n setp.nan.f64 p, %1, %1;\n setp.gt.or.f64 p, %1, %2, p;\n"
                " selp.f64 %0, %1, %2, p;\n}" : "=d"(r) : "d"(a), "d"(b));
        else
            asm("{\n .reg .pred p;\n setp.nan.f64 p, %1, %1;\n setp.lt.or.f64 p, %1, %2, p;\n"
                " selp.f64 %0, %1, %2, p;\n}" : "=d"(r) : "d"(a), "d"(b));
    }
    return r;
}

struct OpMax {
    static constexpr int code = 1;
    static constexpr bool idempotent = true;  // x (+) x == x, bit for bit
    static constexpr bool three = false;
    template <typename T>
    __device__ __forceinline__ static T apply(T a, T b) {
        if constexpr (std::is_integral<T>::value) {
            return a > b ? a : b;
        } else {
            return float_keep_a<T, true>(a, b);
        }
    }
    template <typename T>
    __device__ __forceinline__ static T identity() {
        if constexpr (std::is_same<T, int32_t>::value) return (int32_t)0x80000000u;
        else if constexpr (std::is_same<T, int64_t>::value) return (int64_t)0x8000000000000000ull;
        else return -(T)INFINITY;
    }
};

struct OpMin {
    static constexpr int code = 2;
    static constexpr bool idempotent = true;
    static constexpr bool three = false;
    template <typename T>
    __device__ __forceinline__ static T apply(T a, T b) {
        if constexpr (std::is_integral<T>::value) {
            return a < b ? a : b;
        } else {
            return float_keep_a<T, false>(a, b);  // numpy.minimum, as OpMax
        }
    }
    template <typename T>
    __device__ __forceinline__ static T identity() {
        if constexpr (std::is_same<T, int32_t>::value) return (int32_t)0x7fffffff;
        else if constexpr (std::is_same<T, int64_t>::value) return (int64_t)0x7fffffffffffffffll;
        else return (T)INFINITY;
    }
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
    uint32_t epoch;       // last completed call's tag (0 after init)
    uint32_t done;        // CTAs finished in the current call
    uint32_t error;       // first ls_status error code raised on the device
    uint32_t error_tile;  // tile (or slot) index of that error
    uint32_t pad[28];
};
static_assert(sizeof(Header) == 128, "header is one 128-byte line");

constexpr int kMaxGrid = 4096;

// the latency kernel (lscan_cluster.cuh): 256-thread blocks, one tile each,
// in three geometries chosen from the lab (profiles/r1_cluster_lab.log):
//   small: 4 rows of 16-byte vectors per thread (16 KiB tiles), one cluster
//   mid:   8 rows (32 KiB tiles), several co-resident clusters
//   large: 12 rows (48 KiB tiles), when the mid tiles no longer fit at once
constexpr int kClusterThreads = 256;
constexpr int kClusterGeoms = 4;
constexpr int kClusterRowsSmall = 4, kClusterMinBlocksSmall = 4;
constexpr int kClusterRowsMid = 8, kClusterMinBlocksMid = 2;
constexpr int kClusterRowsLarge = 12, kClusterMinBlocksLarge = 2;
// extra-large: 16 rows (64 KiB tiles, 2 blocks per SM) — reaches 2^22 32-bit /
// 2^21 64-bit elements co-resident, where the persistent kernel's round chain
// costs more than the one-wave cluster exchange
constexpr int kClusterRowsXL = 16, kClusterMinBlocksXL = 2;
constexpr int kClusterMax = 16;  // blocks per cluster (non-portable size; 8 where 16 cannot be scheduled)
constexpr int64_t kClusterMaxBytes = 16ll << 20;  // crossover to the persistent kernel (lab-measured)
constexpr size_t kSlotBase = sizeof(Header) + (size_t)kMaxGrid * 8;

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
    int64_t delay_red_ns;   // debug: reducer sleeps this long on tiles t % 3 == 1 (timing perturbation)
    int64_t delay_scan_ns;  // debug: scanners sleep this long on tiles t % 3 == 2
    int64_t stall_tile;     // debug: this tile never publishes its aggregate (needs a spin budget)
    // ---- multi-GPU (block-cyclic stripes, scan_ws2_kernel<..., MULTI=true>) ----
    int rank, world;               // this GPU's place among `world` GPUs
    uint8_t *xchg;                 // this GPU's exchange region (header + 2 parities of slots)
    uint64_t *const *xchg_peers;   // device array: every GPU's exchange slot base (index = rank)
    int64_t xchg_rounds;           // round capacity per parity
    // ---- x not 16-byte aligned (scan_ws2_kernel<..., SHIFT=true>) ----
    int x_shift;                   // bytes x lies past the 16-byte boundary below it
    int head_n;                    // SHIFT: elements before x / y scanned first (y's 16-byte head)
    int l2_resident;               // x and y together fit in L2: TMA loads evict-normal
};

// cross-GPU exchange region: [Header][parity 0: rounds x world slots][parity 1: ...]
constexpr size_t kXchgSlotBase = 128;

__device__ __forceinline__ void debug_sleep(int64_t ns) {
    while (ns > 0) {
        const unsigned chunk = ns > 100000 ? 100000u : (unsigned)ns;
        __nanosleep(chunk);
        ns -= chunk;
    }
}

// One write-once carry-chain slot per tile / round.  Each 64-bit word holds
// (epoch tag : 32 | 32 value bits); 64-bit values use two words.  A reader
// accepts the slot only when every word carries the current call's tag, so
// the single-copy atomicity of a 64-bit access is the whole handshake.
template <typename T>
struct Slot {
    static constexpr int W = sizeof(T) / 4;  // 64-bit words per slot
    __device__ static void publish(uint64_t *arr, int64_t idx, uint32_t tag, T v) {
        uint64_t *p = arr + idx * W;
        const uint64_t b = (uint64_t)Elem<T>::bits(v);
        slot_st(p, ((uint64_t)tag << 32) | (b & 0xffffffffull));
        if constexpr (W == 2) slot_st(p + 1, ((uint64_t)tag << 32) | (b >> 32));
    }
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
    // system-scope variants for slots written by other GPUs
    __device__ static void publish_sys(uint64_t *arr, int64_t idx, uint32_t tag, T v) {
        uint64_t *p = arr + idx * W;
        const uint64_t b = (uint64_t)Elem<T>::bits(v);
        slot_st_sys(p, ((uint64_t)tag << 32) | (b & 0xffffffffull));
        if constexpr (W == 2) slot_st_sys(p + 1, ((uint64_t)tag << 32) | (b >> 32));
    }
    __device__ static void load_sys(const uint64_t *arr, int64_t idx, uint64_t (&w)[W]) {
        const uint64_t *p = arr + idx * W;
#pragma unroll
        for (int i = 0; i < W; ++i) w[i] = slot_ld_sys(p + i);
    }
};

__device__ __forceinline__ void raise_error(Header *h, uint32_t code, uint32_t where) {
    if (atomicCAS(&h->error, 0u, code) == 0u) h->error_tile = where;
}

// The last CTA to finish records this call's tag as the workspace epoch.
__device__ __forceinline__ void epoch_handover(Header *hdr, uint32_t tag, int grid) {
    const uint32_t old = atom_add_acqrel_u32(&hdr->done, 1u);
    if (old == (uint32_t)grid - 1u) {
        st_relaxed_u32(&hdr->done, 0u);
        st_relaxed_u32(&hdr->epoch, tag);
    }
}

__device__ __forceinline__ uint32_t call_tag(Header *hdr) {
    const uint32_t prev = ld_relaxed_u32(&hdr->epoch);
    return (prev + 1u) == 0u ? 1u : prev + 1u;
}

// ------------------------------------------------------------------------------
template <typename T, int V>
union Regs {
    uint4 q[V];
    T e[V * 16 / sizeof(T)];
};

// 16 bytes of identity elements
template <typename T, typename OP>
__device__ __forceinline__ uint4 identity_vec() {
    Regs<T, 1> r;
#pragma unroll
    for (int e = 0; e < 16 / (int)sizeof(T); ++e) r.e[e] = OP::template identity<T>();
    return r.q[0];
}

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
__device__ __forceinline__ void load_tile_regs(const uint8_t *stage, int tid, Regs<T, V> &r) {
    const int rot = vec_rot<V>(tid);
    const uint32_t base = smem_u32(stage) + (uint32_t)tid * (V * 16);
#pragma unroll
    for (int u = 0; u < V; ++u) r.q[u] = lds128(base + (uint32_t)(((u + rot) & (V - 1)) * 16));
    rotate_left<V>(r.q, (V - rot) & (V - 1));  // r.q[j] now holds vector j
}

template <typename T, int V>
__device__ __forceinline__ void store_tile_regs(uint8_t *stage, int tid, Regs<T, V> &r) {
    const int rot = vec_rot<V>(tid);
    const uint32_t base = smem_u32(stage) + (uint32_t)tid * (V * 16);
    rotate_left<V>(r.q, rot);  // r.q[u] now holds vector (u + rot) mod V
#pragma unroll
    for (int u = 0; u < V; ++u) sts128(base + (uint32_t)(((u + rot) & (V - 1)) * 16), r.q[u]);
}

// v += (the value d lanes down), guarded by the shuffle's own "source lane in
// range" predicate: one SHFL and one predicated add per level (the C++ form
// compiles to SHFL + ISETP/SEL + add).  64-bit values shuffle as two halves
// under the first half's predicate.  IEEE add is commutative, so o + v == v + o.
__device__ __forceinline__ int32_t shfl_up_add(int32_t v, int d) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 t;\n\t"
        "shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n\t@p add.u32 %0, %0, t;\n\t}"
        : "+r"(v)
        : "r"(d));
    return v;
}
__device__ __forceinline__ float shfl_up_add(float v, int d) {
    asm("{\n\t.reg .pred p;\n\t.reg .f32 t;\n\t"
        "shfl.sync.up.b32 t|p, %0, %1, 0, -1;\n\t@p add.rn.f32 %0, %0, t;\n\t}"
        : "+f"(v)
        : "r"(d));
    return v;
}
__device__ __forceinline__ int64_t shfl_up_add(int64_t v, int d) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, tl, th;\n\t.reg .b64 t;\n\t"
        "mov.b64 {lo, hi}, %0;\n\t"
        "shfl.sync.up.b32 tl|p, lo, %1, 0, -1;\n\t"
        "shfl.sync.up.b32 th, hi, %1, 0, -1;\n\t"
        "mov.b64 t, {tl, th};\n\t@p add.u64 %0, %0, t;\n\t}"
        : "+l"(v)
        : "r"(d));
    return v;
}
__device__ __forceinline__ double shfl_up_add(double v, int d) {
    asm("{\n\t.reg .pred p;\n\t.reg .b32 lo, hi, tl, th;\n\t.reg .f64 t;\n\t"
        "mov.b64 {lo, hi}, %0;\n\t"
        "shfl.sync.up.b32 tl|p, lo, %1, 0, -1;\n\t"
        "shfl.sync.up.b32 th, hi, %1, 0, -1;\n\t"
        "mov.b64 t, {tl, th};\n\t@p add.rn.f64 %0, %0, t;\n\t}"
        : "+d"(v)
        : "r"(d));
    return v;
}
#ifndef LS_SHFL_PRED_SCAN
#define LS_SHFL_PRED_SCAN 1
#endif

// Hillis-Steele over the 32 lanes (warp.py:93-109), lower-index operand first.
// PRED: add through shfl_up_add (the latency kernel: i64 2^20 7.41 -> 7.09 us,
// 2^18 5.31 -> 5.12 in the lab; the persistent kernel measured -1 to -2 % with
// it for 64-bit types and keeps the C++ form)
template <typename T, typename OP, bool PRED = false>
__device__ __forceinline__ T warp_inclusive_scan(T v, int lane) {
    if constexpr (PRED && LS_SHFL_PRED_SCAN && OP::code == 0 && !OP::idempotent) {
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) v = shfl_up_add(v, d);
        return v;
    } else {
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T o = __shfl_up_sync(0xffffffffu, v, d);
            // lanes below d get their own value back; an idempotent operator
            // absorbs it, so no lane predicate
            if (OP::idempotent || lane >= d) v = OP::apply(o, v);
        }
        return v;
    }
}

// f32 max / min as one FMNMX: identical to numpy's maximum / minimum on
// operands that are neither zeros nor NaNs (no two distinct bit patterns
// compare equal there, and no NaN to propagate).  The persistent kernel's
// scanners use it for a warp's chunk of a tile holding no zero and no NaN.
// apply3: the three-input FMNMX3 (sm_100) for folds of a lane's elements.
struct OpFastMaxF {
    static constexpr int code = 1;
    static constexpr bool idempotent = true;
    static constexpr bool three = true;
    __device__ __forceinline__ static float apply(float a, float b) { return fmaxf(a, b); }
    __device__ __forceinline__ static float apply3(float a, float b, float c) {
        float r;
        asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
        return r;
    }
};
struct OpFastMinF {
    static constexpr int code = 2;
    static constexpr bool idempotent = true;
    static constexpr bool three = true;
    __device__ __forceinline__ static float apply(float a, float b) { return fminf(a, b); }
    __device__ __forceinline__ static float apply3(float a, float b, float c) {
        float r;
        asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
        return r;
    }
};
// The reducers' f32 max / min: NaN-propagating FMNMX(3).NAN — any NaN makes
// the result a NaN, otherwise it is exact up to the sign of a zero; both
// cases are then re-derived exactly (tile_ties).  Commutative, so lanes agree.
struct OpNanMaxF {
    __device__ __forceinline__ static float apply(float a, float b) {
        float r;
        asm("max.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
        return r;
    }
    __device__ __forceinline__ static float apply3(float a, float b, float c) {
        float r;
        asm("max.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
        return r;
    }
};
struct OpNanMinF {
    __device__ __forceinline__ static float apply(float a, float b) {
        float r;
        asm("min.NaN.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
        return r;
    }
    __device__ __forceinline__ static float apply3(float a, float b, float c) {
        float r;
        asm("min.NaN.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
        return r;
    }
};

// f64 max / min as one DSETP.MAX / .MIN (+ two selects) instead of the exact
// form's two DSETPs: identical to numpy's on operands that are neither zeros
// nor NaNs.  No three-input or NaN-propagating f64 form exists, so the f64
// reducers keep the exact operator (reduce_nan = false).
struct OpFastMaxD {
    static constexpr int code = 1;
    static constexpr bool idempotent = true;
    static constexpr bool three = false;
    __device__ __forceinline__ static double apply(double a, double b) {
        double r;
        asm("max.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
        return r;
    }
};
struct OpFastMinD {
    static constexpr int code = 2;
    static constexpr bool idempotent = true;
    static constexpr bool three = false;
    __device__ __forceinline__ static double apply(double a, double b) {
        double r;
        asm("min.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
        return r;
    }
};

template <typename T, typename OP>
struct ScanFastOp {
    static constexpr bool enabled = false;
    static constexpr bool reduce_nan = false;
    using type = OP;
};
template <>
struct ScanFastOp<float, struct OpMax> {
    static constexpr bool enabled = true;
    static constexpr bool reduce_nan = true;  // the reducers' NaN-propagating FMNMX(3)
    using type = OpFastMaxF;
    using reduce_type = OpNanMaxF;
};
template <>
struct ScanFastOp<float, struct OpMin> {
    static constexpr bool enabled = true;
    static constexpr bool reduce_nan = true;
    using type = OpFastMinF;
    using reduce_type = OpNanMinF;
};
// f64 fast scans: off by default (LS_F64_FAST_SCAN=1 builds them for the
// lab): the chunk test costs 64-bit IADD / IMNMX pairs per element and
// measured slower than the exact DSETP-pair operator it skips
#ifndef LS_F64_FAST_SCAN
#define LS_F64_FAST_SCAN 0
#endif
// f64 NaN-free scans (LS_F64_NANFREE_SCAN): on operands that are not NaN,
// numpy's maximum(a, b) is exactly (a > b) ? a : b — equal operands (+-0
// included) give the right one — so a chunk without NaNs scans with one
// DSETP and two selects per operator and a two-deep dependency chain instead
// of the exact form's NaN test, ordered test and selects.  The chunk test is
// one FADD per element on the high words viewed as f32 (a f64 NaN or infinity
// has all of f32's exponent bits set there, so their sum is not finite)
#ifndef LS_F64_NANFREE_SCAN
#define LS_F64_NANFREE_SCAN 0
#endif
template <bool GT>
struct OpNanFreeD {
    static constexpr int code = GT ? 1 : 2;
    static constexpr bool idempotent = true;
    static constexpr bool three = false;
    __device__ __forceinline__ static double apply(double a, double b) {
        double r;
        if constexpr (GT)
            asm("{\n .reg .pred p;\n setp.gt.f64 p, %1, %2;\n selp.f64 %0, %1, %2, p;\n}" : "=d"(r) : "d"(a), "d"(b));
        else
            asm("{\n .reg .pred p;\n setp.lt.f64 p, %1, %2;\n selp.f64 %0, %1, %2, p;\n}" : "=d"(r) : "d"(a), "d"(b));
        return r;
    }
};
#if LS_F64_FAST_SCAN || LS_F64_NANFREE_SCAN
template <>
struct ScanFastOp<double, struct OpMax> {
    static constexpr bool enabled = true;
    static constexpr bool reduce_nan = false;
#if LS_F64_NANFREE_SCAN
    using type = OpNanFreeD<true>;
#else
    using type = OpFastMaxD;
#endif
};
template <>
struct ScanFastOp<double, struct OpMin> {
    static constexpr bool enabled = true;
    static constexpr bool reduce_nan = false;
#if LS_F64_NANFREE_SCAN
    using type = OpNanFreeD<false>;
#else
    using type = OpFastMinD;
#endif
};
#endif

// A lane's registers hold no zero and no NaN (the fast operators' domain).
// 32-bit words: u = 2 * bits - 1 is 0xffffffff for +-0 and above 0xff000000
// for a NaN, at most 0xfeffffff otherwise (infinities included); 64-bit
// elements the same on the doubled bit pattern (NaN above 0xffe0...0), or,
// for the NaN-free f64 operators, no NaN and no infinity
template <typename T, int V>
__device__ __forceinline__ bool fast_domain(const uint4 (&q)[V]) {
    if constexpr (sizeof(T) == 4) {
        uint32_t mx0 = 0u, mx1 = 0u;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            mx0 = max(mx0, max(q[i].x + q[i].x - 1u, q[i].y + q[i].y - 1u));
            mx1 = max(mx1, max(q[i].z + q[i].z - 1u, q[i].w + q[i].w - 1u));
        }
        return max(mx0, mx1) <= 0xff000000u;
    } else if (LS_F64_NANFREE_SCAN) {
        // no NaN (nor infinity): the high words' f32 sum stays finite
        float s0 = 0.f, s1 = 0.f;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            s0 += __uint_as_float(q[i].y);
            s1 += __uint_as_float(q[i].w);
        }
        return fabsf(s0 + s1) < INFINITY;
    } else {
        unsigned long long mx = 0ull;
#pragma unroll
        for (int i = 0; i < V; ++i) {
            const unsigned long long a = ((unsigned long long)q[i].y << 32) | q[i].x;
            const unsigned long long b = ((unsigned long long)q[i].w << 32) | q[i].z;
            mx = max(mx, max(a + a - 1ull, b + b - 1ull));
        }
        return mx <= 0xffdfffffffffffffull;
    }
}

// Float max/min results depend on the ORDER of equal-comparing operands (-0 /
// +0) and of NaNs: the sequential fold yields the rightmost of the maximal
// elements, or the leftmost NaN.  Every combination of partial results for
// these operators keeps sequence order; add and the integer operators (whose
// equal operands are identical bits) keep their cheaper unordered forms.
template <typename T, typename OP>
__host__ __device__ constexpr bool order_sensitive() {
    return OP::idempotent && std::is_floating_point<T>::value;
}

// the values whose bits an order-free reduction may get wrong
template <typename T>
__device__ __forceinline__ bool tie_class(T v) {
    return v != v || v == (T)0;
}

// fixed xor-butterfly: every lane ends with bit-identical results because
// each level combines a commutative pair.  Order-sensitive operators: levels
// from d = 1 up, the lower lane group always on the left, so every lane holds
// v_0 (+) v_1 (+) ... (+) v_31 in lane order
template <typename T, typename OP>
__device__ __forceinline__ T warp_reduce_fixed(T v) {
    if constexpr (order_sensitive<T, OP>()) {
        const int lane = (int)(threadIdx.x & 31u);
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const T o = __shfl_xor_sync(0xffffffffu, v, d);
            v = (lane & d) ? OP::apply(o, v) : OP::apply(v, o);
        }
    } else {
#pragma unroll
        for (int d = 16; d >= 1; d >>= 1) v = OP::apply(v, __shfl_xor_sync(0xffffffffu, v, d));
    }
    return v;
}

// acc (+) v_0 (+) ... (+) v_31 for lane-strided chunks (lane l holds element
// 32 m + l of chunk m).  Order-free operators accumulate per lane and reduce
// once at the end (finish); order-sensitive ones reduce each chunk in lane
// order into a warp-uniform accumulator
template <typename T, typename OP>
__device__ __forceinline__ T fold_chunk(T acc, T v) {
    if constexpr (order_sensitive<T, OP>()) return OP::apply(acc, warp_reduce_fixed<T, OP>(v));
    else return OP::apply(acc, v);
}
template <typename T, typename OP>
__device__ __forceinline__ T fold_finish(T acc) {
    if constexpr (order_sensitive<T, OP>()) return acc;
    else return warp_reduce_fixed<T, OP>(acc);
}

}  // namespace lscan
