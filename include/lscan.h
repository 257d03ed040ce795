/*
 * lscan.h — C ABI of the B200-native single-pass sum-scan (LightScan,
 * arXiv 1604.04815) that replaces the reference's scan entry point.
 *
 * Reference interface replaced (chainscan 0.1.0, Python):
 *   chained_scan(problem: ScanProblem, config=None) -> ndarray
 *       /root/reference/pkg/src/chainscan/chained.py:316-357
 *   run_algorithm("chained", problem, chain_config)   bench.py:121-147 (:333-334 in file)
 *   ScanProblem (x, op, out; out may alias x)          reference.py:38-58
 *   make_operator("add", i32|i64|f32|f64)              operators.py:111-127
 *   LivenessError / ProtocolViolation                  chained.py:48-53
 *   ChainConfig.spin_budget / corrupt_slot             chained.py:222-224
 *
 * Conventions: plain pointers and sizes only; device pointers are owned by
 * the caller; every device call is stream-ordered and asynchronous (the
 * stream is a cudaStream_t passed as void*, NULL = legacy default stream).
 * Inputs must be 1-D contiguous arrays of the element type; x == y (in
 * place) is allowed, any other overlap of x and y is rejected.  Integer sums
 * wrap modulo 2^width (two's complement), exactly like the reference's
 * np.add under errstate(over="ignore") (operators.py:74-100).
 *
 * Errors are status codes; ls_last_error_detail() returns a thread-local
 * message for the last failing call on the calling thread.
 */
#ifndef LSCAN_H
#define LSCAN_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LS_OK = 0,
    LS_ERR_INVALID_ARG = 1,       /* ShapeError / ValueError (reference.py:50-55, chained.py:227-234) */
    LS_ERR_UNSUPPORTED_DTYPE = 2, /* UnsupportedOperatorError (operators.py:34-47) */
    LS_ERR_CUDA = 3,              /* a CUDA runtime call failed */
    LS_ERR_LIVENESS = 4,          /* LivenessError: debug spin budget exhausted (chained.py:139-144) */
    LS_ERR_PROTOCOL = 5,          /* ProtocolViolation: slot published twice (chained.py:117-118) */
    LS_ERR_WORKSPACE = 6          /* workspace missing / too small / not initialised */
} ls_status;

typedef enum { LS_I32 = 0, LS_I64 = 1, LS_F32 = 2, LS_F64 = 3 } ls_dtype;

/* Scan operators (make_operator, operators.py:111-127): add (identity 0,
 * integers wrap), max (identity = lowest value / -inf), min (highest / +inf).
 * Float max/min are bit-exact to numpy.maximum / numpy.minimum.accumulate,
 * tie rules included: maximum(a, b) = (a > b || isnan(a)) ? a : b, so equal
 * operands give the right one (the sign of a zero result is the rightmost
 * maximal zero's) and a NaN propagates as the leftmost NaN's bits. */
typedef enum { LS_OP_ADD = 0, LS_OP_MAX = 1, LS_OP_MIN = 2 } ls_op;

/* ---- workspace ------------------------------------------------------------
 * The carry-chain buffer (the reference's CommSlots, chained.py:85-150): one
 * write-once slot per data tile plus one per round, epoch-tagged so a call
 * never needs a memset.  Size depends on n and the current device.  A fresh
 * workspace must be zeroed once with ls_workspace_init; after that it can be
 * reused by any number of calls issued in stream order. */
size_t ls_workspace_bytes(ls_dtype dt, int64_t n);
ls_status ls_workspace_init(void *ws, size_t ws_bytes, void *stream);

/* ---- device scans (the hot path) -------------------------------------------
 * y[j] = carry (+) x[0] (+) ... (+) x[j]            (inclusive)
 * y[j] = carry (+) x[0] (+) ... (+) x[j-1]          (exclusive; y[0] = carry,
 *                                                    or the identity)
 * carry_in: nullable device scalar (identity when NULL) — the multi-GPU
 *   carry from lower shards.
 * total_out: nullable device scalar receiving carry (+) x[0] (+) ... (+) x[n-1];
 *   must not alias carry_in.
 * Any element alignment of x and y: 16-byte aligned x with 32-byte aligned y
 * runs at the HBM roofline; other alignments are still one launch (the few
 * elements before y's boundary are folded into the carry inside the kernel,
 * a misaligned x is read through shifted TMA windows) at 84-101 %.
 * Replaces chained_scan (chained.py:316) for the given operator. */
ls_status ls_inclusive_scan(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n,
                            const void *carry_in, void *total_out,
                            void *ws, size_t ws_bytes, void *stream);
ls_status ls_exclusive_scan(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n,
                            const void *carry_in, void *total_out,
                            void *ws, size_t ws_bytes, void *stream);
/* The north-star sum scans: ls_*_scan with LS_OP_ADD. */
ls_status ls_inclusive_sum(ls_dtype dt, const void *x, void *y, int64_t n,
                           const void *carry_in, void *total_out,
                           void *ws, size_t ws_bytes, void *stream);
ls_status ls_exclusive_sum(ls_dtype dt, const void *x, void *y, int64_t n,
                           const void *carry_in, void *total_out,
                           void *ws, size_t ws_bytes, void *stream);

/* The strict left fold: y[j] = y[j-1] (+) x[j] one element after another,
 * the reference's B = 1 path (ChainConfig(b=1), chained.py:290-313), which
 * is bit-identical to sequential_scan (reference.py:61-67) for every
 * operator — float add included, where the parallel scans above associate
 * differently and match only within the envelope.  One CTA runs the
 * dependent chain (about one add latency per element; x streamed in by TMA,
 * y stored by separate warps), so it is an exactness mode, not a fast path.
 * Same conventions as ls_inclusive_scan (any alignment, x == y allowed,
 * carry_in / total_out); exclusive != 0 gives the exclusive form. */
ls_status ls_ordered_scan(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, int exclusive,
                          const void *carry_in, void *total_out, void *stream);

/* total_out = x[0] (+) ... (+) x[n-1] (device scalar; identity for n == 0),
 * deterministic for a given device; the per-shard total of the multi-GPU
 * carry exchange. */
ls_status ls_reduce(ls_op op, ls_dtype dt, const void *x, int64_t n, void *total_out,
                    void *ws, size_t ws_bytes, void *stream);
ls_status ls_reduce_sum(ls_dtype dt, const void *x, int64_t n, void *total_out,
                        void *ws, size_t ws_bytes, void *stream);

/* carry_out = t[0] (+) ... (+) t[rank-1] (identity for rank 0): the fold of
 * the gathered per-rank totals in fixed left-to-right order (SURVEY §8e
 * step 3).  totals is a device array of `count` scalars, carry_out a device
 * scalar. */
ls_status ls_carry_from_totals(ls_op op, ls_dtype dt, const void *totals, int64_t count,
                               int64_t rank, void *carry_out, void *stream);

/* ---- multi-GPU, block-cyclic (fused exchange) --------------------
 * `world` GPUs (one process each) scan one global array distributed
 * block-cyclically, the reference's cyclic block ownership (chained.py:264-287)
 * lifted from workers to GPUs: every GPU holds n_local elements (the same n_local
 * on every GPU) cut into stripes of G tiles (G = the launch grid, identical on
 * every GPU), and the global order is stripe 0 of GPU 0, stripe 0 of GPU 1, ...,
 * stripe 1 of GPU 0, ...  One kernel per GPU does everything: stripe aggregates
 * are pushed into every GPU's exchange region (peer memory over NVLink,
 * system-scope tagged words) as soon as the data lands, and one warp per GPU
 * folds them into the global round chain — no host synchronisation, no NCCL.
 * xchg: this GPU's exchange region (ls_xchg_bytes, zeroed once with
 *   ls_workspace_init before ANY GPU's first call — barrier after init);
 * xchg_peers: device array of `world` pointers, entry g = GPU g's exchange
 *   region as mapped in this process (entry rank = xchg);
 * grid > 0 caps the CTAs (equal on every GPU), 0 = the device's capacity.
 * total_out receives the GLOBAL total.  All GPUs must make the same sequence
 * of calls.  A watchdog is always armed (a large default probe budget, or the
 * ls_debug_config budget): a peer that died or never launches its half of a
 * call turns into LS_ERR_LIVENESS in the workspace instead of a hang.  These
 * calls never synchronise on it (all GPUs of a call must be in flight
 * together): read the outcome with ls_workspace_error. */
size_t ls_xchg_bytes(ls_dtype dt, int world, int64_t n_local);
ls_status ls_inclusive_scan_multi(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n_local,
                                  const void *carry_in, void *total_out, void *ws, size_t ws_bytes,
                                  int rank, int world, void *xchg, size_t xchg_bytes,
                                  void *const *xchg_peers, int grid, void *stream);
ls_status ls_exclusive_scan_multi(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n_local,
                                  const void *carry_in, void *total_out, void *ws, size_t ws_bytes,
                                  int rank, int world, void *xchg, size_t xchg_bytes,
                                  void *const *xchg_peers, int grid, void *stream);
/* Device memory that can be shared with peer processes (cudaMalloc'd), and
 * CUDA IPC handles (64 bytes) to map it in another process. */
ls_status ls_device_alloc(size_t bytes, void **out);
ls_status ls_device_free(void *ptr);
ls_status ls_ipc_get_handle(void *dev_ptr, void *handle_out);
ls_status ls_ipc_open(const void *handle, void **dev_ptr_out);
ls_status ls_ipc_close(void *dev_ptr);

/* ---- host-buffer entry (what chained_scan(problem) does with numpy arrays) --
 * x and y are HOST pointers (pinned or pageable; y may equal x).  The array
 * is streamed through the device in chunks with copy-in, scan and copy-out
 * overlapped on three streams, the carry chained on the device between
 * chunks.  Blocks until y is complete.  device < 0 = current device. */
ls_status ls_scan_host(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n,
                       int exclusive, int device);
/* ls_scan_host with flags: LS_HOST_EXCLUSIVE, LS_HOST_ORDERED (every chunk
 * through ls_ordered_scan, the carry chained between chunks: the whole array
 * is one strict left fold — ChainConfig(b=1)). */
#define LS_HOST_EXCLUSIVE 1
#define LS_HOST_ORDERED 2
ls_status ls_scan_host_ex(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n,
                          int flags, int device);
ls_status ls_inclusive_sum_host(ls_dtype dt, const void *x, void *y, int64_t n,
                                int exclusive, int device);

/* ---- debug hooks (ChainConfig.spin_budget / corrupt_slot, chained.py:222-224)
 * spin_budget > 0 arms a device watchdog: a look-back that probes a slot more
 * than spin_budget times records LS_ERR_LIVENESS in the workspace instead of
 * hanging.  corrupt_block >= 0 makes that tile publish the identity as its
 * aggregate (fault injection; the output is wrong only after that tile).
 * With either armed, or protocol_checks != 0, every device call synchronises
 * its stream and reports the workspace error word as its status.
 * Process-wide; (0, -1, 0) disarms. */
ls_status ls_debug_config(int64_t spin_budget, int64_t corrupt_block, int protocol_checks);

/* Timing perturbation for race testing (the device analogue of the
 * reference's randomised on_block delays, test_chained.py:239-256): the
 * reducer warp sleeps reducer_delay_ns on tiles t % 3 == 1 and one scanner
 * warp sleeps scanner_delay_ns on tiles t % 3 == 2.  Results must not change.
 * stall_tile >= 0 makes that tile never publish its aggregate — a real stall
 * of the chain (test_chained.py:259-272); it is honoured only while a spin
 * budget is armed, so the watchdog turns it into LS_ERR_LIVENESS.
 * Process-wide; (0, 0, -1) disarms. */
ls_status ls_debug_perturb(int64_t reducer_delay_ns, int64_t scanner_delay_ns, int64_t stall_tile);

/* Kernel selection for testing: 0 = automatic (small n on the one-cluster
 * latency kernel, the rest on the persistent chain), 1 = never use the
 * cluster kernel, 2 = use it whenever n fits one cluster (even while debug
 * hooks are armed, which it ignores).  Process-wide. */
ls_status ls_debug_force_path(int path);

/* Slot handshake stress (the reference's acceptance criterion 4,
 * test_acceptance.py:146-196, on the device): one writer publishes `count`
 * slots of dtype dt while reader_ctas x 128 threads re-read them; out[0] =
 * reads, out[1] = torn pairs seen (must be 0), out[2] = published slots seen
 * unpublished again by the same reader (must be 0).  Synchronous. */
ls_status ls_debug_slot_stress(ls_dtype dt, int64_t count, int reader_ctas, int64_t stats_out[3]);

/* Reads and clears the device error word of a workspace (synchronises). */
ls_status ls_workspace_error(void *ws, size_t ws_bytes, void *stream);

/* ---- introspection ---------------------------------------------------------- */
const char *ls_status_string(ls_status s);
const char *ls_last_error_detail(void);
int ls_abi_version(void);
/* Launch geometry the scan uses on the current device for dt:
 * out[0] = persistent CTAs (grid), out[1] = threads per CTA, out[2] = elements
 * per tile, out[3] = pipeline stages, out[4] = resident CTAs per SM,
 * out[5] = SM count. */
ls_status ls_query_config(ls_dtype dt, int64_t n, int64_t out[6]);
/* The multi-GPU kernel (ls_*_scan_multi) for n_local elements per GPU:
 * out[0] = its default grid (CTAs per GPU), out[1] = elements per tile.  The
 * block-cyclic stripe is grid * tile elements (GPU g's stripe k is global
 * stripe k * world + g). */
ls_status ls_query_multi_config(ls_dtype dt, int64_t n_local, int64_t out[2]);
/* The latency kernel (small and mid n) on the current device: out[0] =
 * blocks per cluster (0 = unavailable), out[1] = elements per block (one
 * tile each) while n fits one cluster, out[2] = co-resident clusters of the
 * mid geometry, out[3] = largest n the kernel takes, out[4] = elements per
 * block of the mid geometry, out[5] = largest n on mid tiles (beyond it,
 * tiles of 3 * out[1] elements).  A scan of n <= out[3] elements (debug
 * hooks disarmed) is one launch: carries travel through distributed shared
 * memory inside a cluster and through epoch-tagged workspace slots between
 * clusters. */
ls_status ls_query_cluster(ls_dtype dt, int64_t out[6]);
/* Number of kernel launches this process has issued through the library. */
int64_t ls_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* LSCAN_H */
