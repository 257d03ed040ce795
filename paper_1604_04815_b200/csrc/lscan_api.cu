// lscan_api.cu — the C ABI (include/lscan.h): argument checking, launch
// geometry, the workspace protocol and the debug hooks.
//
// The reference entry point this replaces is chained_scan(problem, config)
// (chainscan/chained.py:316-357); see include/lscan.h for the per-function
// mapping.  Kernels are instantiated per element type in lscan_inst_*.cu.
//
// Kernel selection per call (scan_impl):
//   n <= cluster_limit (~10 MiB), debug hooks off  -> scan_cluster_kernel (any alignment)
//   x 16-byte, y (16 * vw)-byte aligned             -> scan_ws2_kernel (TMA, persistent)
//   otherwise, n >= 2^20                            -> one launch of scan_ws2_kernel (x lands
//                                                      16-byte aligned after y's head) or of
//                                                      ws2<SHIFT> (shifted x windows); y's head
//                                                      folded into the carry in the kernel
//   otherwise                                       -> scan_generic_kernel
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstddef>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <deque>
#include <vector>

#include "lscan.h"
#include "lscan_dispatch.h"

using namespace lscan;

namespace lscan {
thread_local std::string g_detail;
void set_detail(const std::string &msg) { g_detail = msg; }
}  // namespace lscan

namespace {

std::atomic<int64_t> g_launches{0};

struct DebugCfg {
    int64_t spin_budget = 0;
    int64_t corrupt = -1;
    int protocol = 0;
    int64_t delay_red_ns = 0;
    int64_t delay_scan_ns = 0;
    int64_t stall_tile = -1;
    int force_path = 0;  // ls_debug_force_path
    bool armed() const { return spin_budget > 0 || corrupt >= 0 || protocol != 0; }
};
std::mutex g_dbg_mu;
DebugCfg g_dbg;

DebugCfg debug_snapshot() {
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    return g_dbg;
}

ls_status fail(ls_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_detail = buf;
    return s;
}

ls_status cuda_fail(cudaError_t e, const char *what) {
    return fail(LS_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
}

#define LS_CUDA(call, what)                                \
    do {                                                   \
        cudaError_t e_ = (call);                           \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

// below this size a misaligned input the latency kernel does not take (debug
// hooks armed, forced persistent path) runs on the generic kernel
constexpr int64_t kSplitMinElems = 1 << 20;

// default look-back / exchange probe budget of the multi-GPU kernel
constexpr int64_t kMultiSpinBudget = int64_t(1) << 28;

// LSCAN_NO_COOP=1: plain launches (lab measurement of the cooperative-launch
// cost).  The grid never exceeds the co-resident capacity either way.
bool cooperative_launch() {
    static const bool coop = [] {
        const char *e = getenv("LSCAN_NO_COOP");
        return !(e && e[0] == '1');
    }();
    return coop;
}

// LSCAN_NO_CLUSTER=1: small arrays take the persistent kernel too (lab
// comparison of the two latency paths)
bool cluster_path_enabled() {
    static const bool on = [] {
        const char *e = getenv("LSCAN_NO_CLUSTER");
        return !(e && e[0] == '1');
    }();
    return on;
}

// LSCAN_NO_PDL=1: launch the latency kernel without programmatic dependent
// launch (lab A/B of the overlap between back-to-back calls)
bool pdl_enabled() {
    static const bool on = [] {
        const char *e = getenv("LSCAN_NO_PDL");
        return !(e && e[0] == '1');
    }();
    return on;
}

bool valid_dtype(ls_dtype dt) { return dt >= LS_I32 && dt <= LS_F64; }
bool valid_op(ls_op op) { return op >= LS_OP_ADD && op <= LS_OP_MIN; }

int elem_size(ls_dtype dt) {
    switch (dt) {
    case LS_I32: case LS_F32: return 4;
    case LS_I64: case LS_F64: return 8;
    default: return 0;
    }
}

const DtypeKernels &K(ls_dtype dt) {
    switch (dt) {
    case LS_I64: return kernels_i64();
    case LS_F32: return kernels_f32();
    case LS_F64: return kernels_f64();
    default: return kernels_i32();
    }
}

int64_t tile_elems(ls_dtype dt, bool fast) {
    return (fast ? K(dt).scan[0][0][1].tile_bytes : kGenTileBytes) / elem_size(dt);
}
int64_t num_tiles(ls_dtype dt, int64_t n, bool fast) {
    const int64_t te = tile_elems(dt, fast);
    return (n + te - 1) / te;
}
// the workspace must fit whichever path has the smaller tiles
int64_t max_tiles(ls_dtype dt, int64_t n) { return std::max(num_tiles(dt, n, true), num_tiles(dt, n, false)); }

struct DevState {
    bool init = false;
    int sms = 0;
    int occ[4][kNumOps][2][2] = {};  // resident CTAs per SM [dtype][op][excl][fast]
    int occ_multi[4][kNumOps][2] = {};
    int occ_shift[4][kNumOps][2] = {};
    int reduce_occ[4][kNumOps] = {};
    int cluster_max = 0;          // largest schedulable cluster of the latency kernel (0: path off)
    int xl_cluster = 0;           // cluster size of the extra-large geometry (the one placing most blocks)
    int cluster_capacity[kClusterGeoms] = {};  // co-resident clusters of that size per geometry (min over instances)
    int64_t l2_bytes = 0;
};
std::mutex g_dev_mu;
std::deque<DevState> g_dev;  // deque: growing it never moves the states other threads hold

// LSCAN_NO_XL=1: no extra-large cluster geometry (lab A/B)
bool xl_geometry_enabled() {
    static const bool on = [] {
        const char *e = getenv("LSCAN_NO_XL");
        return !(e && e[0] == '1');
    }();
    return on;
}

ls_status device_state(DevState **out) {
    int dev = 0;
    LS_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
    DevState &d = g_dev[dev];
    if (!d.init) {
        LS_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
        int l2 = 0;
        LS_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev), "L2 size");
        d.l2_bytes = l2;
        for (int dt = 0; dt < 4; ++dt) {
            const DtypeKernels &k = K((ls_dtype)dt);
            for (int op = 0; op < kNumOps; ++op) {
                for (int ex = 0; ex < 2; ++ex)
                    for (int fa = 0; fa < 2; ++fa) {
                        const Launch &L = k.scan[op][ex][fa];
                        LS_CUDA(cudaFuncSetAttribute((const void *)L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                     (int)L.smem),
                                "cudaFuncSetAttribute(max dynamic smem)");
                        int occ = 0;
                        LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)L.fn, L.threads,
                                                                              L.smem),
                                "occupancy query");
                        if (occ < 1) return fail(LS_ERR_CUDA, "scan kernel cannot be resident (smem %zu B)", L.smem);
                        d.occ[dt][op][ex][fa] = occ;
                    }
                for (int ex = 0; ex < 2; ++ex) {
                    const Launch &L = k.multi[op][ex];
                    LS_CUDA(cudaFuncSetAttribute((const void *)L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)L.smem),
                            "cudaFuncSetAttribute(max dynamic smem)");
                    int occm = 0;
                    LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occm, (const void *)L.fn, L.threads, L.smem),
                            "occupancy query");
                    if (occm < 1) return fail(LS_ERR_CUDA, "multi scan kernel cannot be resident");
                    d.occ_multi[dt][op][ex] = occm;
                }
                for (int ex = 0; ex < 2; ++ex) {
                    const Launch &L = k.shift[op][ex];
                    LS_CUDA(cudaFuncSetAttribute((const void *)L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)L.smem),
                            "cudaFuncSetAttribute(max dynamic smem)");
                    int occs = 0;
                    LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occs, (const void *)L.fn, L.threads, L.smem),
                            "occupancy query");
                    d.occ_shift[dt][op][ex] = occs;
                }
                for (int ex = 0; ex < 2; ++ex)
                    LS_CUDA(cudaFuncSetAttribute((const void *)k.ordered[op][ex].fn,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k.ordered[op][ex].smem),
                            "cudaFuncSetAttribute(max dynamic smem)");
                int occ = 0;
                LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k.reduce_fn[op], kReduceThreads, 0),
                        "occupancy");
                d.reduce_occ[dt][op] = std::max(occ, 1);
                for (int ex = 0; ex < 2; ++ex)
                    for (int g = 0; g < kClusterGeoms; ++g)
                        LS_CUDA(cudaFuncSetAttribute((const void *)k.cluster[op][ex][g].fn,
                                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1),
                                "cudaFuncSetAttribute(non-portable cluster size)");
            }
        }
        // the latency path needs a whole cluster co-resident: 16 blocks where
        // the GPCs allow it, else the portable 8; and for several clusters,
        // how many fit at once (the minimum over every instance)
        d.cluster_max = 0;
        int caps[2][kClusterGeoms];  // [16, 8][geometry]: co-resident clusters (min over every instance)
        const int sizes[2] = {kClusterMax, 8};
        for (int si = 0; si < 2; ++si) {
            const int c = sizes[si];
            int *cap = caps[si];
            for (int g = 0; g < kClusterGeoms; ++g) cap[g] = 1 << 30;
            for (int g = 0; g < kClusterGeoms; ++g)
                for (int dt = 0; dt < 4; ++dt)
                    for (int op = 0; op < kNumOps; ++op)
                        for (int ex = 0; ex < 2; ++ex) {
                            const Launch &L = K((ls_dtype)dt).cluster[op][ex][g];
                            cudaLaunchConfig_t cfg = {};
                            cfg.gridDim = dim3((unsigned)c);
                            cfg.blockDim = dim3((unsigned)L.threads);
                            cudaLaunchAttribute attr[1];
                            attr[0].id = cudaLaunchAttributeClusterDimension;
                            attr[0].val.clusterDim.x = (unsigned)c;
                            attr[0].val.clusterDim.y = 1;
                            attr[0].val.clusterDim.z = 1;
                            cfg.attrs = attr;
                            cfg.numAttrs = 1;
                            int nc = 0;
                            if (cudaOccupancyMaxActiveClusters(&nc, (const void *)L.fn, &cfg) != cudaSuccess) {
                                (void)cudaGetLastError();
                                nc = 0;
                            }
                            cap[g] = std::min(cap[g], nc);
                        }
        }
        for (int si = 0; si < 2; ++si) {
            const int *cap = caps[si];
            // the extra-large geometry is optional (its span is 0 without it)
            if (cap[0] >= 1 && cap[1] >= 1 && cap[2] >= 1) {
                d.cluster_max = sizes[si];
                for (int g = 0; g < kClusterGeoms; ++g) d.cluster_capacity[g] = cap[g];
                // extra-large tiles: whichever cluster size places the most blocks
                // at once (GPC packing can favour 8-block clusters there)
                d.xl_cluster = sizes[si];
                for (int sj = si; sj < 2; ++sj)
                    if (caps[sj][3] * sizes[sj] > d.cluster_capacity[3] * d.xl_cluster) {
                        d.xl_cluster = sizes[sj];
                        d.cluster_capacity[3] = caps[sj][3];
                    }
                if (!xl_geometry_enabled()) d.cluster_capacity[3] = 0;
                break;
            }
        }
        d.init = true;
    }
    *out = &d;
    return LS_OK;
}

ls_status check_ws_header(const void *ws, size_t ws_bytes, size_t need) {
    if (!ws) return fail(LS_ERR_WORKSPACE, "workspace is NULL");
    if (((uintptr_t)ws & 127u) != 0) return fail(LS_ERR_WORKSPACE, "workspace must be 128-byte aligned");
    if (ws_bytes < need) return fail(LS_ERR_WORKSPACE, "workspace too small: %zu < %zu bytes", ws_bytes, need);
    return LS_OK;
}

ls_status read_device_error(void *ws, cudaStream_t s, bool clear) {
    Header h;
    LS_CUDA(cudaStreamSynchronize(s), "cudaStreamSynchronize");
    LS_CUDA(cudaMemcpy(&h, ws, sizeof(h), cudaMemcpyDeviceToHost), "read workspace header");
    if (h.error != 0) {
        const uint32_t code = h.error, where = h.error_tile;
        if (clear) {
            uint32_t zero[2] = {0, 0};
            LS_CUDA(cudaMemcpy((uint8_t *)ws + offsetof(Header, error), zero, sizeof zero, cudaMemcpyHostToDevice),
                    "clear workspace error");
        }
        if (code == LS_ERR_LIVENESS)
            return fail(LS_ERR_LIVENESS, "spin budget exhausted in the look-back of tile %u", where);
        if (code == LS_ERR_PROTOCOL) return fail(LS_ERR_PROTOCOL, "slot %u written twice", where);
        return fail((ls_status)code, "device error %u at %u", code, where);
    }
    return LS_OK;
}

bool ranges_overlap(const void *a, const void *b, size_t bytes) {
    const uintptr_t x = (uintptr_t)a, y = (uintptr_t)b;
    return x < y + bytes && y < x + bytes;
}

ls_status identity_fill(ls_op op, ls_dtype dt, void *dst, const void *carry_in, cudaStream_t s) {
    // total of an empty scan: the carry, else the operator's identity (the
    // carry fold over zero ranks writes exactly that, stream-ordered)
    if (carry_in) {
        LS_CUDA(cudaMemcpyAsync(dst, carry_in, elem_size(dt), cudaMemcpyDeviceToDevice, s), "copy carry");
        return LS_OK;
    }
    K(dt).launch_carry(op, nullptr, 0, dst, s);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LS_CUDA(cudaGetLastError(), "identity fill");
    return LS_OK;
}

// Small and mid n: one tile per block, clusters of up to d.cluster_max
// blocks (carries through DSMEM), several clusters co-resident by a
// cooperative launch (cluster aggregates through epoch-tagged slots).
// Geometry g: 0 = small tiles (n fits one cluster of them), 1 = mid tiles
// (while their clusters fit at once), 2 = large tiles, 3 = extra-large tiles
// (beyond the large ones' co-resident capacity).
int cluster_size(const DevState &d, int g) { return g == 3 ? d.xl_cluster : d.cluster_max; }

int64_t cluster_span(const DevState &d, ls_dtype dt, int g) {  // elements the geometry covers
    const int64_t te = K(dt).cluster[0][0][g].tile_bytes / elem_size(dt);
    return te * cluster_size(d, g) * (g == 0 ? 1 : d.cluster_capacity[g]);
}

int cluster_geometry(const DevState &d, ls_dtype dt, int64_t n) {
    static const int forced = [] {  // LSCAN_CLUSTER_GEOM=1|2|3: lab A/B of the multi-cluster geometries
        const char *e = getenv("LSCAN_CLUSTER_GEOM");
        return e ? atoi(e) : 0;
    }();
    if (n <= cluster_span(d, dt, 0)) return 0;
    if (forced >= 1 && forced < kClusterGeoms && n <= cluster_span(d, dt, forced)) return forced;
    if (n <= cluster_span(d, dt, 1)) return 1;
    return n <= cluster_span(d, dt, 2) ? 2 : 3;
}

ls_status launch_cluster(const DevState &d, ls_op op, ls_dtype dt, const void *x, void *y, int64_t n,
                         const void *carry_in, void *total_out, void *ws, cudaStream_t s, bool excl) {
    const int g = cluster_geometry(d, dt, n);
    const Launch &L = K(dt).cluster[op][excl][g];
    const int64_t te = L.tile_bytes / elem_size(dt);
    const int64_t tiles = (n + te - 1) / te;
    const int C = (int)std::min<int64_t>(tiles, cluster_size(d, g));
    const int64_t clusters = (tiles + C - 1) / C;
    ScanParams p{};
    p.x = x;
    p.y = y;
    p.n = n;
    p.carry_in = carry_in;
    p.total_out = total_out;
    p.ws = static_cast<uint8_t *>(ws);
    p.num_tiles = tiles;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(clusters * C));
    cfg.blockDim = dim3((unsigned)L.threads);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    if (clusters > 1) {
        // several clusters wait on each other's aggregates: all must be resident
        attr[1].id = cudaLaunchAttributeCooperative;
        attr[1].val.cooperative = 1;
    } else {
        // one cluster: may launch early behind the previous kernel (PDL); the
        // kernel's griddepcontrol.wait keeps the data dependency
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = (clusters > 1 || pdl_enabled()) ? 2 : 1;
    LS_CUDA(cudaLaunchKernelEx(&cfg, L.fn, p), "cluster scan kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return LS_OK;
}

// largest n the cluster kernel takes: one cluster of small tiles always;
// mid / large tiles up to their co-resident capacity and the measured
// crossover with the persistent kernel (LSCAN_CLUSTER_MAX_BYTES overrides it
// for labs)
int64_t cluster_limit(const DevState &d, ls_dtype dt) {
    static const int64_t max_bytes = [] {
        const char *e = getenv("LSCAN_CLUSTER_MAX_BYTES");
        return e ? std::max<int64_t>(0, atoll(e)) : kClusterMaxBytes;
    }();
    const int64_t coresident =
        std::max(std::max(cluster_span(d, dt, 1), cluster_span(d, dt, 2)), cluster_span(d, dt, 3));
    return std::max(cluster_span(d, dt, 0), std::min(coresident, max_bytes / elem_size(dt)));
}

bool use_cluster(const DevState &d, ls_dtype dt, int64_t n, const DebugCfg &dbg) {
    // the debug hooks (watchdog, corrupt / stalled tiles, perturbation) live
    // in the persistent kernel's carry chain: keep those calls on it
    if (d.cluster_max == 0 || dbg.force_path == 1) return false;
    if (dbg.force_path != 2 && (!cluster_path_enabled() || dbg.armed() || dbg.delay_red_ns > 0 ||
                                dbg.delay_scan_ns > 0 || dbg.stall_tile >= 0))
        return false;
    return n <= cluster_limit(d, dt);
}

// Evict-normal TMA loads when the call's traffic fits well inside L2 (x then
// stays for a caller that reads it again); LSCAN_L2_POLICY=first|normal
// overrides for labs
bool l2_policy_normal(const DevState &d, int64_t bytes) {
    static const int mode = [] {
        const char *e = getenv("LSCAN_L2_POLICY");
        if (!e) return 0;
        return strcmp(e, "first") == 0 ? 1 : (strcmp(e, "normal") == 0 ? 2 : 0);
    }();
    if (mode) return mode == 2;
    return bytes <= d.l2_bytes * 3 / 4;
}

// One kernel launch of the fast (TMA, 16-byte aligned) or generic path.
// x_shift > 0: the shifted-window kernel over a misaligned x (x_shift bytes
// past a 16-byte boundary; y aligned), after folding the head_n elements
// just before x / y into the carry (and storing them)
ls_status launch_scan(const DevState &d, ls_op op, ls_dtype dt, const void *x, void *y, int64_t n,
                      const void *carry_in, void *total_out, void *ws, cudaStream_t s, bool excl, bool fast,
                      const DebugCfg &dbg, int x_shift = 0, int head_n = 0) {
    const Launch &L = x_shift ? K(dt).shift[op][excl] : K(dt).scan[op][excl][fast];
    // tiles of this kernel's own geometry (the shifted-window kernel's may
    // differ from the aligned one's; every geometry's tile is at least the
    // generic kernel's, which sizes the workspace)
    const int64_t te = L.tile_bytes / elem_size(dt);
    const int64_t M = (n + te - 1) / te;
    const int64_t cap = (int64_t)(x_shift ? d.occ_shift[dt][op][excl] : d.occ[dt][op][excl][fast]) * d.sms;
    int G = (int)std::min<int64_t>(M, cap);
    static const int balanced = [] {
        const char *e = getenv("LSCAN_BALANCED_GRID");  // lab switch
        return e ? atoi(e) : 0;
    }();
    if (balanced && G > 0) {
        // the fewest CTAs that keep the same number of rounds: every CTA gets
        // the same tile count
        const int64_t rounds = (M + G - 1) / G;
        G = (int)((M + rounds - 1) / rounds);
    }
    ScanParams p{};
    p.x = x;
    p.y = y;
    p.n = n;
    p.carry_in = carry_in;
    p.total_out = total_out;
    p.ws = static_cast<uint8_t *>(ws);
    p.num_tiles = M;
    p.spin_budget = dbg.spin_budget;
    p.corrupt_tile = dbg.corrupt;
    p.protocol_checks = dbg.protocol;
    p.delay_red_ns = dbg.delay_red_ns;
    p.delay_scan_ns = dbg.delay_scan_ns;
    // a stalled tile without a watchdog would hang the chain forever
    p.stall_tile = dbg.spin_budget > 0 ? dbg.stall_tile : -1;
    p.x_shift = x_shift;
    p.head_n = head_n;
    p.l2_resident = l2_policy_normal(d, 2 * n * (int64_t)elem_size(dt)) ? 1 : 0;

    // Cooperative launch: the driver refuses a grid that cannot be fully
    // co-resident — the deadlock-freedom precondition of the persistent
    // chain (chainscan/schedsim.py's invariant).
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3((unsigned)L.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (cooperative_launch()) {
        attr[na].id = cudaLaunchAttributeCooperative;
        attr[na++].val.cooperative = 1;
    }
    if (fast && pdl_enabled()) {
        // the TMA kernel waits on griddepcontrol before touching global
        // memory, so it may launch behind the previous kernel's tail
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    LS_CUDA(cudaLaunchKernelEx(&cfg, L.fn, p), "scan kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return LS_OK;
}

ls_status scan_impl(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in, void *total_out,
                    void *ws, size_t ws_bytes, void *stream, bool excl) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (!valid_op(op)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported operator code %d", (int)op);
    const int es = elem_size(dt);
    if (n < 0) return fail(LS_ERR_INVALID_ARG, "n must be >= 0, got %lld", (long long)n);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n > 0 && (!x || !y)) return fail(LS_ERR_INVALID_ARG, "x and y must be non-NULL for n > 0");
    if (((uintptr_t)x % es) || ((uintptr_t)y % es))
        return fail(LS_ERR_INVALID_ARG, "x and y must be aligned to the element size (%d)", es);
    if (x != y && n > 0 && ranges_overlap(x, y, (size_t)n * es))
        return fail(LS_ERR_INVALID_ARG, "x and y overlap without being identical (only exact in-place is allowed)");
    if (total_out && carry_in && total_out == carry_in)
        return fail(LS_ERR_INVALID_ARG, "total_out must not alias carry_in");
    if (n == 0) return total_out ? identity_fill(op, dt, total_out, carry_in, s) : LS_OK;
    ls_status st = check_ws_header(ws, ws_bytes, ls_workspace_bytes(dt, n));
    if (st != LS_OK) return st;
    DevState *d = nullptr;
    if ((st = device_state(&d)) != LS_OK) return st;
    const DebugCfg dbg = debug_snapshot();

    bool launched = false;
    if (use_cluster(*d, dt, n, dbg)) {
        // a cluster grid the GPU cannot place right now (its GPCs held by
        // other work) fails at launch without side effects: the persistent
        // kernel takes the call instead
        st = launch_cluster(*d, op, dt, x, y, n, carry_in, total_out, ws, s, excl);
        launched = st == LS_OK;
        if (!launched && dbg.force_path != 2) {
            (void)cudaGetLastError();
            st = LS_OK;
        }
    }
    if (!launched && st == LS_OK) {
        // the persistent kernel tiles y on (16 * vw)-byte boundaries (its
        // 256-bit stores need 32); the head before y's first boundary is folded
        // into the carry inside the kernel, so every alignment is one launch:
        // x then lands 16-byte aligned (TMA tiles) or not (shifted windows)
        const unsigned ya = 16u * (unsigned)K(dt).ws2_vw[op];
        const unsigned yoff = (unsigned)((uintptr_t)y % ya);
        const int64_t head = yoff ? (int64_t)((ya - yoff) / (unsigned)es) : 0;
        const uint8_t *xb = static_cast<const uint8_t *>(x) + head * es;
        uint8_t *yb = static_cast<uint8_t *>(y) + head * es;
        const int xs = (int)((uintptr_t)xb & 15u);
        if (head == 0 && xs == 0) {
            st = launch_scan(*d, op, dt, x, y, n, carry_in, total_out, ws, s, excl, true, dbg);
        } else if (n >= kSplitMinElems && xs == 0) {
            st = launch_scan(*d, op, dt, xb, yb, n - head, carry_in, total_out, ws, s, excl, true, dbg, 0, (int)head);
        } else if (n >= kSplitMinElems && d->occ_shift[dt][op][excl] > 0) {
            st = launch_scan(*d, op, dt, xb, yb, n - head, carry_in, total_out, ws, s, excl, true, dbg, xs, (int)head);
        } else {
            st = launch_scan(*d, op, dt, x, y, n, carry_in, total_out, ws, s, excl, false, dbg);
        }
    }
    if (st != LS_OK) return st;
    if (dbg.armed()) return read_device_error(ws, s, true);
    return LS_OK;
}

}  // namespace

// ======================================================================= ABI ==
extern "C" {

int ls_abi_version(void) { return 1; }

const char *ls_status_string(ls_status s) {
    switch (s) {
    case LS_OK: return "LS_OK";
    case LS_ERR_INVALID_ARG: return "LS_ERR_INVALID_ARG";
    case LS_ERR_UNSUPPORTED_DTYPE: return "LS_ERR_UNSUPPORTED_DTYPE";
    case LS_ERR_CUDA: return "LS_ERR_CUDA";
    case LS_ERR_LIVENESS: return "LS_ERR_LIVENESS";
    case LS_ERR_PROTOCOL: return "LS_ERR_PROTOCOL";
    case LS_ERR_WORKSPACE: return "LS_ERR_WORKSPACE";
    }
    return "LS_ERR_UNKNOWN";
}

const char *ls_last_error_detail(void) { return g_detail.c_str(); }

int64_t ls_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

size_t ls_workspace_bytes(ls_dtype dt, int64_t n) {
    if (!valid_dtype(dt) || n < 0) return 0;
    const int64_t M = std::max<int64_t>(max_tiles(dt, n), 1);
    const size_t sw = elem_size(dt) == 4 ? 8 : 16;
    const size_t bytes = kSlotBase + 2 * (size_t)M * sw;
    return (bytes + 255) & ~(size_t)255;
}

ls_status ls_workspace_init(void *ws, size_t ws_bytes, void *stream) {
    if (!ws || ws_bytes < sizeof(Header)) return fail(LS_ERR_WORKSPACE, "workspace NULL or smaller than its header");
    LS_CUDA(cudaMemsetAsync(ws, 0, ws_bytes, static_cast<cudaStream_t>(stream)), "workspace memset");
    return LS_OK;
}

ls_status ls_inclusive_scan(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in,
                            void *total_out, void *ws, size_t ws_bytes, void *stream) {
    return scan_impl(op, dt, x, y, n, carry_in, total_out, ws, ws_bytes, stream, false);
}

ls_status ls_exclusive_scan(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in,
                            void *total_out, void *ws, size_t ws_bytes, void *stream) {
    return scan_impl(op, dt, x, y, n, carry_in, total_out, ws, ws_bytes, stream, true);
}

ls_status ls_inclusive_sum(ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in, void *total_out,
                           void *ws, size_t ws_bytes, void *stream) {
    return scan_impl(LS_OP_ADD, dt, x, y, n, carry_in, total_out, ws, ws_bytes, stream, false);
}

ls_status ls_exclusive_sum(ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in, void *total_out,
                           void *ws, size_t ws_bytes, void *stream) {
    return scan_impl(LS_OP_ADD, dt, x, y, n, carry_in, total_out, ws, ws_bytes, stream, true);
}

ls_status ls_ordered_scan(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, int exclusive,
                          const void *carry_in, void *total_out, void *stream) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (!valid_op(op)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported operator code %d", (int)op);
    const int es = elem_size(dt);
    if (n < 0) return fail(LS_ERR_INVALID_ARG, "n must be >= 0, got %lld", (long long)n);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n > 0 && (!x || !y)) return fail(LS_ERR_INVALID_ARG, "x and y must be non-NULL for n > 0");
    if (((uintptr_t)x % es) || ((uintptr_t)y % es))
        return fail(LS_ERR_INVALID_ARG, "x and y must be aligned to the element size (%d)", es);
    if (x != y && n > 0 && ranges_overlap(x, y, (size_t)n * es))
        return fail(LS_ERR_INVALID_ARG, "x and y overlap without being identical (only exact in-place is allowed)");
    if (total_out && carry_in && total_out == carry_in)
        return fail(LS_ERR_INVALID_ARG, "total_out must not alias carry_in");
    if (n == 0) return total_out ? identity_fill(op, dt, total_out, carry_in, s) : LS_OK;
    DevState *d = nullptr;
    ls_status st = device_state(&d);
    if (st != LS_OK) return st;
    const Launch &L = K(dt).ordered[op][exclusive ? 1 : 0];
    ScanParams p{};
    p.x = x;
    p.y = y;
    p.n = n;
    p.carry_in = carry_in;
    p.total_out = total_out;
    L.fn<<<1, L.threads, L.smem, s>>>(p);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LS_CUDA(cudaGetLastError(), "ordered scan kernel launch");
    return LS_OK;
}

ls_status ls_reduce(ls_op op, ls_dtype dt, const void *x, int64_t n, void *total_out, void *ws, size_t ws_bytes,
                    void *stream) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (!valid_op(op)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported operator code %d", (int)op);
    if (n < 0) return fail(LS_ERR_INVALID_ARG, "n must be >= 0");
    if (!total_out) return fail(LS_ERR_INVALID_ARG, "total_out must be non-NULL");
    const int es = elem_size(dt);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) return identity_fill(op, dt, total_out, nullptr, s);
    if (!x || ((uintptr_t)x % es)) return fail(LS_ERR_INVALID_ARG, "x NULL or misaligned");
    ls_status st = check_ws_header(ws, ws_bytes, kSlotBase);
    if (st != LS_OK) return st;
    DevState *d = nullptr;
    if ((st = device_state(&d)) != LS_OK) return st;
    const int64_t per_cta = (int64_t)kReduceThreads * (32 / es) * 4;
    int64_t grid = std::min<int64_t>((n + per_cta - 1) / per_cta, (int64_t)d->reduce_occ[dt][op] * d->sms);
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, kMaxGrid));
    // the head of x (read last by the reverse sweep) stays in L2 for a scan
    // of the same array right behind: up to half of L2
    const int64_t keep = std::min<int64_t>(n * es, (int64_t)d->l2_bytes / 2);
    K(dt).launch_reduce(op, x, n, total_out, ws, (int)grid, keep, s);
    // float max/min add the tie fix-up kernel (lscan_generic.cuh)
    const bool ties = op != LS_OP_ADD && (dt == LS_F32 || dt == LS_F64);
    g_launches.fetch_add(ties ? 2 : 1, std::memory_order_relaxed);
    LS_CUDA(cudaGetLastError(), "reduce kernel launch");
    return LS_OK;
}

ls_status ls_reduce_sum(ls_dtype dt, const void *x, int64_t n, void *total_out, void *ws, size_t ws_bytes,
                        void *stream) {
    return ls_reduce(LS_OP_ADD, dt, x, n, total_out, ws, ws_bytes, stream);
}

ls_status ls_carry_from_totals(ls_op op, ls_dtype dt, const void *totals, int64_t count, int64_t rank,
                               void *carry_out, void *stream) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (!valid_op(op)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported operator code %d", (int)op);
    if (!totals || !carry_out || count < 1 || rank < 0 || rank >= count)
        return fail(LS_ERR_INVALID_ARG, "bad totals/carry_out/count/rank");
    K(dt).launch_carry(op, totals, rank, carry_out, static_cast<cudaStream_t>(stream));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LS_CUDA(cudaGetLastError(), "carry kernel launch");
    return LS_OK;
}

// tiles of the multi-GPU kernel (its own geometry, MultiCfg)
int64_t multi_tiles(ls_dtype dt, int64_t n) {
    const int64_t te = K(dt).multi[0][0].tile_bytes / elem_size(dt);
    return (n + te - 1) / te;
}

size_t ls_xchg_bytes(ls_dtype dt, int world, int64_t n_local) {
    if (!valid_dtype(dt) || world < 1 || n_local < 0) return 0;
    const int64_t rounds = std::max<int64_t>(multi_tiles(dt, n_local), 1);  // rounds <= tiles
    const size_t sw = elem_size(dt) == 4 ? 8 : 16;
    const size_t bytes = kXchgSlotBase + 2 * (size_t)rounds * (size_t)world * sw;
    return (bytes + 255) & ~(size_t)255;
}

static ls_status scan_multi_impl(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in,
                                 void *total_out, void *ws, size_t ws_bytes, int rank, int world, void *xchg,
                                 size_t xchg_bytes, void *const *peers, int grid, void *stream, bool excl) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (!valid_op(op)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported operator code %d", (int)op);
    if (world < 1 || world > 32 || rank < 0 || rank >= world) return fail(LS_ERR_INVALID_ARG, "bad rank/world");
    if (n < 1 || !x || !y) return fail(LS_ERR_INVALID_ARG, "multi-GPU scan needs n >= 1 and device buffers");
    if ((((uintptr_t)x | (uintptr_t)y) & 15u) != 0)
        return fail(LS_ERR_INVALID_ARG, "multi-GPU scan needs 16-byte aligned x and y");
    const int es = elem_size(dt);
    if (x != y && ranges_overlap(x, y, (size_t)n * es))
        return fail(LS_ERR_INVALID_ARG, "x and y overlap without being identical");
    if (!xchg || !peers || xchg_bytes < ls_xchg_bytes(dt, world, n) || ((uintptr_t)xchg & 127u))
        return fail(LS_ERR_WORKSPACE, "exchange region missing, misaligned or too small");
    ls_status st = check_ws_header(ws, ws_bytes, ls_workspace_bytes(dt, n));
    if (st != LS_OK) return st;
    DevState *d = nullptr;
    if ((st = device_state(&d)) != LS_OK) return st;
    const Launch &L = K(dt).multi[op][excl];
    const int64_t M = multi_tiles(dt, n);
    const int64_t cap = (int64_t)d->occ_multi[dt][op][excl] * d->sms;
    int64_t G = std::min<int64_t>(M, cap);
    if (grid > 0) {
        if (grid > cap) return fail(LS_ERR_INVALID_ARG, "grid %d exceeds co-resident capacity %lld", grid, (long long)cap);
        G = std::min<int64_t>(M, grid);
    }
    const DebugCfg dbg = debug_snapshot();
    ScanParams p{};
    p.x = x;
    p.y = y;
    p.n = n;
    p.carry_in = carry_in;
    p.total_out = total_out;
    p.ws = static_cast<uint8_t *>(ws);
    p.num_tiles = M;
    // the watchdog is always armed here: a peer GPU that died or never
    // launches its half of the call must become LS_ERR_LIVENESS in the
    // workspace (ls_workspace_error), not a hang of every other GPU.  The
    // default budget is large (each probe sleeps; ~30 s or more of waiting)
    p.spin_budget = dbg.spin_budget > 0 ? dbg.spin_budget : kMultiSpinBudget;
    p.corrupt_tile = dbg.corrupt;
    p.protocol_checks = dbg.protocol;
    p.delay_red_ns = dbg.delay_red_ns;
    p.delay_scan_ns = dbg.delay_scan_ns;
    p.stall_tile = dbg.spin_budget > 0 ? dbg.stall_tile : -1;
    p.rank = rank;
    p.world = world;
    p.xchg = static_cast<uint8_t *>(xchg);
    p.xchg_peers = reinterpret_cast<uint64_t *const *>(peers);
    // the parity halves' stride is the region's fixed capacity (in rounds),
    // never this call's round count: consecutive calls with different n (the
    // short last chunk of scan_host) must keep their halves apart
    p.xchg_rounds = (int64_t)((xchg_bytes - kXchgSlotBase) / (2 * (size_t)world * (es == 4 ? 8 : 16)));
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3((unsigned)L.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    // programmatic dependent launch as for the single-GPU kernel: the wait
    // precedes every global access, and the exchange region's parity double
    // buffer already separates consecutive calls across GPUs
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    LS_CUDA(cudaLaunchKernelEx(&cfg, L.fn, p), "multi scan kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    // no debug synchronisation here: the GPUs of one call must all be in
    // flight together; read the error word afterwards (ls_workspace_error)
    return LS_OK;
}

ls_status ls_inclusive_scan_multi(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n_local,
                                  const void *carry_in, void *total_out, void *ws, size_t ws_bytes, int rank,
                                  int world, void *xchg, size_t xchg_bytes, void *const *xchg_peers, int grid,
                                  void *stream) {
    return scan_multi_impl(op, dt, x, y, n_local, carry_in, total_out, ws, ws_bytes, rank, world, xchg, xchg_bytes,
                           xchg_peers, grid, stream, false);
}

ls_status ls_exclusive_scan_multi(ls_op op, ls_dtype dt, const void *x, void *y, int64_t n_local,
                                  const void *carry_in, void *total_out, void *ws, size_t ws_bytes, int rank,
                                  int world, void *xchg, size_t xchg_bytes, void *const *xchg_peers, int grid,
                                  void *stream) {
    return scan_multi_impl(op, dt, x, y, n_local, carry_in, total_out, ws, ws_bytes, rank, world, xchg, xchg_bytes,
                           xchg_peers, grid, stream, true);
}

ls_status ls_device_alloc(size_t bytes, void **out) {
    if (!out) return fail(LS_ERR_INVALID_ARG, "out is NULL");
    LS_CUDA(cudaMalloc(out, bytes), "cudaMalloc");
    return LS_OK;
}

ls_status ls_device_free(void *ptr) {
    LS_CUDA(cudaFree(ptr), "cudaFree");
    return LS_OK;
}

ls_status ls_ipc_get_handle(void *dev_ptr, void *handle_out) {
    if (!dev_ptr || !handle_out) return fail(LS_ERR_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    LS_CUDA(cudaIpcGetMemHandle(&h, dev_ptr), "cudaIpcGetMemHandle");
    memcpy(handle_out, &h, sizeof h);
    return LS_OK;
}

ls_status ls_ipc_open(const void *handle, void **dev_ptr_out) {
    if (!handle || !dev_ptr_out) return fail(LS_ERR_INVALID_ARG, "NULL argument");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof h);
    LS_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    return LS_OK;
}

ls_status ls_ipc_close(void *dev_ptr) {
    LS_CUDA(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
    return LS_OK;
}

ls_status ls_debug_config(int64_t spin_budget, int64_t corrupt_block, int protocol_checks) {
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    g_dbg.spin_budget = spin_budget > 0 ? spin_budget : 0;
    g_dbg.corrupt = corrupt_block >= 0 ? corrupt_block : -1;
    g_dbg.protocol = protocol_checks ? 1 : 0;
    return LS_OK;
}

ls_status ls_debug_perturb(int64_t reducer_delay_ns, int64_t scanner_delay_ns, int64_t stall_tile) {
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    g_dbg.stall_tile = stall_tile >= 0 ? stall_tile : -1;
    g_dbg.delay_red_ns = reducer_delay_ns > 0 ? reducer_delay_ns : 0;
    g_dbg.delay_scan_ns = scanner_delay_ns > 0 ? scanner_delay_ns : 0;
    return LS_OK;
}

ls_status ls_debug_force_path(int path) {
    if (path < 0 || path > 2) return fail(LS_ERR_INVALID_ARG, "path must be 0, 1 or 2");
    std::lock_guard<std::mutex> lk(g_dbg_mu);
    g_dbg.force_path = path;
    return LS_OK;
}

ls_status ls_debug_slot_stress(ls_dtype dt, int64_t count, int reader_ctas, int64_t stats_out[3]) {
    if (!valid_dtype(dt) || count < 128 || reader_ctas < 1 || reader_ctas > 1024 || !stats_out)
        return fail(LS_ERR_INVALID_ARG, "bad stress arguments");
    const size_t sw = elem_size(dt) == 4 ? 8 : 16;
    void *buf = nullptr;
    const size_t bytes = 64 + (size_t)count * sw;
    LS_CUDA(cudaMalloc(&buf, bytes), "cudaMalloc");
    ls_status st = LS_OK;
    do {
        cudaError_t e = cudaMemset(buf, 0, bytes);
        if (e != cudaSuccess) { st = cuda_fail(e, "memset"); break; }
        unsigned long long *stats = static_cast<unsigned long long *>(buf);
        int *done = reinterpret_cast<int *>(static_cast<uint8_t *>(buf) + 32);
        uint64_t *slots = reinterpret_cast<uint64_t *>(static_cast<uint8_t *>(buf) + 64);
        // the stress needs the writer and the readers co-resident: a few CTAs only
        K(dt).launch_stress(slots, count, 0x5eedu, done, stats, reader_ctas, 0);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { st = cuda_fail(e, "slot stress kernel"); break; }
        unsigned long long h[3];
        e = cudaMemcpy(h, stats, sizeof h, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) { st = cuda_fail(e, "read stress stats"); break; }
        for (int i = 0; i < 3; ++i) stats_out[i] = (int64_t)h[i];
    } while (0);
    cudaFree(buf);
    return st;
}

ls_status ls_workspace_error(void *ws, size_t ws_bytes, void *stream) {
    ls_status st = check_ws_header(ws, ws_bytes, kSlotBase);
    if (st != LS_OK) return st;
    return read_device_error(ws, static_cast<cudaStream_t>(stream), true);
}

ls_status ls_query_config(ls_dtype dt, int64_t n, int64_t out[6]) {
    if (!valid_dtype(dt) || !out || n < 0) return fail(LS_ERR_INVALID_ARG, "bad arguments");
    DevState *d = nullptr;
    ls_status st = device_state(&d);
    if (st != LS_OK) return st;
    const Launch &L = K(dt).scan[0][0][1];
    const int occ = d->occ[dt][0][0][1];
    const int64_t M = num_tiles(dt, n, true);
    out[0] = std::min<int64_t>(std::max<int64_t>(M, 1), (int64_t)occ * d->sms);
    out[1] = L.threads;
    out[2] = tile_elems(dt, true);
    out[3] = L.stages;
    out[4] = occ;
    out[5] = d->sms;
    return LS_OK;
}

ls_status ls_query_multi_config(ls_dtype dt, int64_t n_local, int64_t out[2]) {
    if (!valid_dtype(dt) || !out || n_local < 0) return fail(LS_ERR_INVALID_ARG, "bad arguments");
    DevState *d = nullptr;
    ls_status st = device_state(&d);
    if (st != LS_OK) return st;
    out[0] = std::min<int64_t>(std::max<int64_t>(multi_tiles(dt, n_local), 1), (int64_t)d->occ_multi[dt][0][0] * d->sms);
    out[1] = K(dt).multi[0][0].tile_bytes / elem_size(dt);
    return LS_OK;
}

ls_status ls_query_cluster(ls_dtype dt, int64_t out[6]) {
    if (!valid_dtype(dt) || !out) return fail(LS_ERR_INVALID_ARG, "bad arguments");
    DevState *d = nullptr;
    ls_status st = device_state(&d);
    if (st != LS_OK) return st;
    out[0] = cluster_path_enabled() ? d->cluster_max : 0;
    out[1] = K(dt).cluster[0][0][0].tile_bytes / elem_size(dt);
    out[2] = cluster_path_enabled() ? d->cluster_capacity[1] : 0;
    out[3] = cluster_path_enabled() ? cluster_limit(*d, dt) : 0;
    out[4] = K(dt).cluster[0][0][1].tile_bytes / elem_size(dt);
    out[5] = cluster_path_enabled() ? cluster_span(*d, dt, 1) : 0;
    return LS_OK;
}

}  // extern "C"
