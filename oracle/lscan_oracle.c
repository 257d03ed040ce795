/*
 * lscan_oracle.c — CPU restatement of the reference scan path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library, and
 * only as the checker or the timed CPU baseline — never as the product path.
 *
 * Reference (Python + numpy, /root/reference/pkg/src/chainscan):
 *   sequential fold   reference.py:61-67  -> operators.py:87-94
 *                     (np.add.accumulate with dtype pinned, errstate(over=ignore):
 *                      a strict left fold in the element type; integers wrap
 *                      modulo 2^width, which C gets through unsigned arithmetic)
 *   chained scan      chained.py:316-357 (entry), :264-287 (cyclic worker loop),
 *                     :237-249 (vectorized block scan: local accumulate, then
 *                     combine(left, seg)), :153-172 (inter_block_comm: block 0
 *                     publishes its reduction, block i waits on slot i-1 and
 *                     publishes left (+) reduction), :290-313 (B == 1 path: carry
 *                     prepended, bit-identical to the sequential fold),
 *                     :85-150 (CommSlots: write-once value/flag pairs)
 *
 * The chained restatement runs on real POSIX threads with C11 release/acquire
 * flags instead of per-slot mutexes (the reference needs the mutex only
 * because CPython cannot publish a (value, flag) pair atomically; here the
 * value is written before the flag is released, so a reader that acquires
 * the flag sees the value: the same transactional guarantee).
 *
 * dtype codes match include/lscan.h: 0 = i32, 1 = i64, 2 = f32, 3 = f64.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <sched.h>
#include <stdatomic.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_I32 = 0, OR_I64 = 1, OR_F32 = 2, OR_F64 = 3 };
enum { OR_OK = 0, OR_BAD_ARG = 1, OR_BAD_DTYPE = 2, OR_NOMEM = 3 };

/* ---- per-type strict left folds ------------------------------------------ */
/* inclusive: y[j] = (((c + x0) + x1) + ... + xj); without a carry the fold
 * starts from x0 itself, exactly like ufunc.accumulate (operators.py:91-94).
 * exclusive: y[j] = fold of everything strictly before j (identity / carry at
 * j = 0) — the derived mode of SURVEY §8a row a19. */
#define DEFINE_FOLD(NAME, T, ACC)                                               \
    static T NAME(const T *x, T *y, int64_t n, int has_carry, T carry,          \
                  int exclusive) {                                              \
        ACC acc = (ACC)carry;                                                   \
        int64_t j = 0;                                                          \
        if (!has_carry && n > 0) {                                              \
            if (exclusive) { y[0] = (T)0; acc = (ACC)x[0]; }                    \
            else { acc = (ACC)x[0]; y[0] = (T)acc; }                            \
            j = 1;                                                              \
        }                                                                       \
        if (exclusive) {                                                        \
            for (; j < n; ++j) { ACC v = (ACC)x[j]; y[j] = (T)acc; acc = acc + v; } \
        } else {                                                                \
            for (; j < n; ++j) { acc = acc + (ACC)x[j]; y[j] = (T)acc; }        \
        }                                                                       \
        return (T)acc;                                                          \
    }

DEFINE_FOLD(fold_i32, int32_t, uint32_t)
DEFINE_FOLD(fold_i64, int64_t, uint64_t)
DEFINE_FOLD(fold_f32, float, float)
DEFINE_FOLD(fold_f64, double, double)

static int elem_size(int dt) {
    switch (dt) {
    case OR_I32: case OR_F32: return 4;
    case OR_I64: case OR_F64: return 8;
    default: return 0;
    }
}

/* Generic dispatch of one fold over a slice; carry/total are scalars of the
 * element type passed by pointer (carry may be NULL). */
static void fold_any(int dt, const void *x, void *y, int64_t n,
                     const void *carry, void *total, int exclusive) {
    switch (dt) {
    case OR_I32: {
        int32_t c = carry ? *(const int32_t *)carry : 0;
        int32_t t = fold_i32((const int32_t *)x, (int32_t *)y, n, carry != 0, c, exclusive);
        if (total) *(int32_t *)total = t;
        break;
    }
    case OR_I64: {
        int64_t c = carry ? *(const int64_t *)carry : 0;
        int64_t t = fold_i64((const int64_t *)x, (int64_t *)y, n, carry != 0, c, exclusive);
        if (total) *(int64_t *)total = t;
        break;
    }
    case OR_F32: {
        float c = carry ? *(const float *)carry : 0.0f;
        float t = fold_f32((const float *)x, (float *)y, n, carry != 0, c, exclusive);
        if (total) *(float *)total = t;
        break;
    }
    case OR_F64: {
        double c = carry ? *(const double *)carry : 0.0;
        double t = fold_f64((const double *)x, (double *)y, n, carry != 0, c, exclusive);
        if (total) *(double *)total = t;
        break;
    }
    }
}

/* sequential_scan (reference.py:61-67).  carry_in seeds the fold (the chunked
 * oracle for arrays larger than host RAM carries it across chunks the way
 * _scan_single does, chained.py:299-313); total_out receives the inclusive
 * total of carry (+) x[0..n).  n == 0 leaves y untouched (reference.py:64-65)
 * and reports the carry (or identity) as the total. */
int oracle_sequential_scan(int dt, const void *x, void *y, int64_t n,
                           int exclusive, const void *carry_in, void *total_out) {
    int es = elem_size(dt);
    if (!es) return OR_BAD_DTYPE;
    if (n < 0 || (n > 0 && (!x || !y))) return OR_BAD_ARG;
    if (n == 0) {
        if (total_out) {
            if (carry_in) memcpy(total_out, carry_in, (size_t)es);
            else memset(total_out, 0, (size_t)es);
        }
        return OR_OK;
    }
    fold_any(dt, x, y, n, carry_in, total_out, exclusive);
    return OR_OK;
}

/* Sum of x[0..n) as a left fold (the per-shard total of the multi-GPU carry
 * exchange). */
int oracle_reduce_sum(int dt, const void *x, int64_t n, void *total_out) {
    int es = elem_size(dt);
    if (!es) return OR_BAD_DTYPE;
    if (n < 0 || !total_out || (n > 0 && !x)) return OR_BAD_ARG;
    switch (dt) {
    case OR_I32: { uint32_t a = 0; const int32_t *p = x; for (int64_t j = 0; j < n; ++j) a += (uint32_t)p[j]; *(int32_t *)total_out = (int32_t)a; break; }
    case OR_I64: { uint64_t a = 0; const int64_t *p = x; for (int64_t j = 0; j < n; ++j) a += (uint64_t)p[j]; *(int64_t *)total_out = (int64_t)a; break; }
    case OR_F32: { float a = 0; const float *p = x; if (n) a = p[0]; for (int64_t j = 1; j < n; ++j) a = a + p[j]; *(float *)total_out = a; break; }
    case OR_F64: { double a = 0; const double *p = x; if (n) a = p[0]; for (int64_t j = 1; j < n; ++j) a = a + p[j]; *(double *)total_out = a; break; }
    }
    return OR_OK;
}

/* ---- chained scan on real threads (chained.py:316-357) --------------------- */

typedef struct {
    /* CommSlots (chained.py:85-150): value row + flag row per slot.  The
     * 128-byte padding of the reference (VALUE_PAD_BYTES, chained.py:38) is
     * kept so neighbouring slots never share a cache line on the host. */
    unsigned char *values;   /* count * 128 bytes, value at offset 0 */
    _Atomic int64_t *flags;  /* count * 16 int64 (128 B stride), flag at [16*i] */
    int64_t count;
} slots_t;

typedef struct {
    int dt, es, b, exclusive;
    const unsigned char *x;
    unsigned char *y;
    int64_t n, L, m, corrupt_block;
    slots_t *slots;
    _Atomic int violation;
} chain_job_t;

typedef struct { chain_job_t *job; int wid; } chain_arg_t;

static void slot_store(slots_t *s, int64_t i, const void *v, int es, _Atomic int *violation) {
    /* write-once discipline (chained.py:114-120): second publish is a
     * ProtocolViolation; recorded, not raised, on the C side */
    if (atomic_load_explicit(&s->flags[16 * i], memory_order_relaxed)) {
        atomic_store(violation, 1);
        return;
    }
    memcpy(s->values + 128 * i, v, (size_t)es);
    atomic_store_explicit(&s->flags[16 * i], 1, memory_order_release);
}

static void slot_wait(slots_t *s, int64_t i, void *out, int es) {
    /* spin-then-yield (SpinPolicy default, chained.py:60-82, :131-150) */
    int probes = 0;
    while (!atomic_load_explicit(&s->flags[16 * i], memory_order_acquire)) {
        if (++probes >= 1024) sched_yield();
    }
    memcpy(out, s->values + 128 * i, (size_t)es);
}

/* combine(left, seg) over a block: seg[j] = left (+) seg[j]  (chained.py:248-249) */
static void fold_left_into(int dt, const void *left, void *seg, int64_t len) {
    switch (dt) {
    case OR_I32: { uint32_t l = *(const uint32_t *)left; uint32_t *p = seg; for (int64_t j = 0; j < len; ++j) p[j] = l + p[j]; break; }
    case OR_I64: { uint64_t l = *(const uint64_t *)left; uint64_t *p = seg; for (int64_t j = 0; j < len; ++j) p[j] = l + p[j]; break; }
    case OR_F32: { float l = *(const float *)left; float *p = seg; for (int64_t j = 0; j < len; ++j) p[j] = l + p[j]; break; }
    case OR_F64: { double l = *(const double *)left; double *p = seg; for (int64_t j = 0; j < len; ++j) p[j] = l + p[j]; break; }
    }
}

static void add_scalar(int dt, const void *a, const void *b, void *out) {
    switch (dt) {
    case OR_I32: *(uint32_t *)out = *(const uint32_t *)a + *(const uint32_t *)b; break;
    case OR_I64: *(uint64_t *)out = *(const uint64_t *)a + *(const uint64_t *)b; break;
    case OR_F32: *(float *)out = *(const float *)a + *(const float *)b; break;
    case OR_F64: *(double *)out = *(const double *)a + *(const double *)b; break;
    }
}

static void *chain_worker(void *p) {
    chain_arg_t *a = p;
    chain_job_t *j = a->job;
    int es = j->es;
    unsigned char zero[8] = {0}, red[8], left[8], total[8];
    /* cyclic ownership: worker wid owns blocks wid, wid+B, ... in ascending
     * order (chained.py:270) */
    for (int64_t i = a->wid; i < j->m; i += j->b) {
        int64_t lo = i * j->L, hi = lo + j->L < j->n ? lo + j->L : j->n;
        const unsigned char *xs = j->x + lo * es;
        unsigned char *ys = j->y + lo * es;
        /* local accumulate straight into the output slice (chained.py:241-243) */
        fold_any(j->dt, xs, ys, hi - lo, NULL, red, 0);
        /* inter_block_comm (chained.py:153-172) */
        if (i == 0) {
            memcpy(left, zero, 8);
            memcpy(total, red, 8);
        } else {
            slot_wait(j->slots, i - 1, left, es);
            add_scalar(j->dt, left, red, total);
        }
        slot_store(j->slots, i, i == j->corrupt_block ? zero : total, es, &j->violation);
        if (i) fold_left_into(j->dt, left, ys, hi - lo);
    }
    return NULL;
}

/* chained_scan(problem, ChainConfig(b=workers, geometry with block_len L)).
 * workers is capped at the block count (chained.py:337); B == 1 takes the
 * fused single-worker path, which is bit-identical to the sequential fold
 * (chained.py:290-313).  corrupt_block >= 0 publishes the identity for that
 * block (ChainConfig.corrupt_slot, chained.py:224/:171).  In-place (y == x)
 * is safe for the same reason as in the reference (chained.py:319-321).
 * Returns 0, or 4 when a slot was published twice (ProtocolViolation). */
int oracle_chained_scan(int dt, const void *x, void *y, int64_t n,
                        int64_t block_len, int workers, int64_t corrupt_block) {
    int es = elem_size(dt);
    if (!es) return OR_BAD_DTYPE;
    if (n < 0 || block_len < 1 || workers < 1 || (n > 0 && (!x || !y))) return OR_BAD_ARG;
    if (n == 0) return OR_OK;
    int64_t m = (n + block_len - 1) / block_len;
    int64_t b64 = workers < m ? workers : m;
    int b = (int)(b64 < 1 ? 1 : b64);
    slots_t slots;
    slots.count = m;
    slots.values = calloc((size_t)m, 128);
    slots.flags = calloc((size_t)m * 16, sizeof(int64_t));
    if (!slots.values || !slots.flags) { free(slots.values); free((void *)slots.flags); return OR_NOMEM; }
    chain_job_t job = {dt, es, b, 0, x, y, n, block_len, m, corrupt_block, &slots, 0};
    if (b == 1) {
        unsigned char carry[8];
        for (int64_t i = 0; i < m; ++i) {
            int64_t lo = i * block_len, hi = lo + block_len < n ? lo + block_len : n;
            fold_any(dt, (const unsigned char *)x + lo * es, (unsigned char *)y + lo * es,
                     hi - lo, i ? carry : NULL, carry, 0);
            unsigned char zero[8] = {0};
            slot_store(&slots, i, i == corrupt_block ? zero : carry, es, &job.violation);
            /* the B == 1 path keeps its own carry: a poisoned slot does not
             * change its output (chained.py:312-313) */
        }
    } else {
        pthread_t *th = malloc(sizeof(pthread_t) * (size_t)b);
        chain_arg_t *args = malloc(sizeof(chain_arg_t) * (size_t)b);
        if (!th || !args) { free(th); free(args); free(slots.values); free((void *)slots.flags); return OR_NOMEM; }
        for (int w = 0; w < b; ++w) {
            args[w].job = &job;
            args[w].wid = w;
            pthread_create(&th[w], NULL, chain_worker, &args[w]);
        }
        for (int w = 0; w < b; ++w) pthread_join(th[w], NULL);
        free(th);
        free(args);
    }
    int rc = atomic_load(&job.violation) ? 4 : OR_OK;
    free(slots.values);
    free((void *)slots.flags);
    return rc;
}

int oracle_abi_version(void) { return 1; }
