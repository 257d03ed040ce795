// lscan_api.cu — the C ABI (include/lscan.h): argument checking, launch
// geometry, workspace protocol, debug hooks, and the host-buffer pipeline
// that streams numpy-resident arrays through the device scan.
//
// The reference entry point this replaces is chained_scan(problem, config)
// (chainscan/chained.py:316-357); see include/lscan.h for the per-function
// mapping.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "lscan.h"
#include "lscan_kernels.cuh"
#include "lscan_scan_ws2.cuh"

using namespace lscan;

namespace lscan {
thread_local std::string g_detail;
void set_detail(const std::string &msg) { g_detail = msg; }
}  // namespace lscan

namespace {

// ---------------------------------------------------------------- tuning --
// Hot path (16-byte aligned x and y): the warp-specialised kernel with
// register-resident results (scan_ws2_kernel) — 8 scanner warps + producer +
// reducer + look-back warps, one 32 KiB tile of x per iteration, six-deep TMA
// ring (192 KiB smem) -> one CTA per SM.  Chosen from the lab sweep in
// profiles/r1_lab_ws2.json (810 Gelem/s i32, ~99.5% of the measured copy).
// Generic path (any element alignment): the sequential kernel with plain
// loads/stores through a two-tile staging buffer.
template <int ES>
struct FastCfg;
// 32-bit elements: 8 scanner warps, 32 KiB tiles (8192 elements), 6 stages
template <>
struct FastCfg<4> {
    static constexpr int kScanWarps = 8, kTileBytes = 32768, kStages = 6;
};
// 64-bit elements: 12 scanner warps, 48 KiB tiles (6144 elements), 4 stages
// (profiles/r1_lab_ws2_wide.json: 398 Gelem/s vs 370 for the 32-bit shape)
template <>
struct FastCfg<8> {
    static constexpr int kScanWarps = 12, kTileBytes = 49152, kStages = 4;
};
constexpr int kThreads = 512;  // generic path
constexpr int kGenTileBytes = 32768;
constexpr int kGenStages = 2;
constexpr int kReduceThreads = 512;

std::atomic<int64_t> g_launches{0};

struct DebugCfg {
    int64_t spin_budget = 0;
    int64_t corrupt = -1;
    int protocol = 0;
    int64_t delay_red_ns = 0;
    int64_t delay_scan_ns = 0;
    int64_t stall_tile = -1;
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

#define LS_CUDA(call, what)                              \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, what); \
    } while (0)

int elem_size(ls_dtype dt) {
    switch (dt) {
    case LS_I32: case LS_F32: return 4;
    case LS_I64: case LS_F64: return 8;
    default: return 0;
    }
}

int fast_tile_bytes(int es) { return es == 4 ? FastCfg<4>::kTileBytes : FastCfg<8>::kTileBytes; }
int64_t tile_elems(ls_dtype dt, bool fast) {
    return (fast ? fast_tile_bytes(elem_size(dt)) : kGenTileBytes) / elem_size(dt);
}
int64_t num_tiles(ls_dtype dt, int64_t n, bool fast) {
    const int64_t te = tile_elems(dt, fast);
    return (n + te - 1) / te;
}
// the workspace must fit the path with the smaller tiles
int64_t max_tiles(ls_dtype dt, int64_t n) { return std::max(num_tiles(dt, n, true), num_tiles(dt, n, false)); }

size_t gen_smem(int es) {
    return (size_t)kGenStages * kGenTileBytes + (size_t)kGenStages * 8 + (size_t)(2 * (kThreads / 32) + 1) * es + 16;
}

// ----------------------------------------------------- kernel dispatch --
using ScanFn = void (*)(const ScanParams);

struct Launch {
    ScanFn fn;
    int threads;
    size_t smem;
};

template <typename T>
Launch pick_typed(bool excl, bool fast) {
    using C = FastCfg<sizeof(T)>;
    if (fast)
        return {excl ? &scan_ws2_kernel<T, C::kScanWarps, C::kTileBytes, C::kStages, true>
                     : &scan_ws2_kernel<T, C::kScanWarps, C::kTileBytes, C::kStages, false>,
                (C::kScanWarps + 3) * 32, scan_ws2_smem_bytes<T, C::kScanWarps, C::kTileBytes, C::kStages>()};
    return {excl ? &scan_kernel<T, kThreads, kGenTileBytes, kGenStages, true, false>
                 : &scan_kernel<T, kThreads, kGenTileBytes, kGenStages, false, false>,
            kThreads, gen_smem(sizeof(T))};
}

Launch pick_scan(ls_dtype dt, bool excl, bool fast) {
    switch (dt) {
    case LS_I32: return pick_typed<uint32_t>(excl, fast);
    case LS_I64: return pick_typed<uint64_t>(excl, fast);
    case LS_F32: return pick_typed<float>(excl, fast);
    case LS_F64: return pick_typed<double>(excl, fast);
    }
    return {nullptr, 0, 0};
}

struct DevState {
    bool init = false;
    int sms = 0;
    // resident CTAs per SM for [dtype][excl][tma]
    int occ[4][2][2] = {};
    int reduce_occ[4] = {};
};
std::mutex g_dev_mu;
std::vector<DevState> g_dev;

ls_status device_state(DevState **out) {
    int dev = 0;
    LS_CUDA(cudaGetDevice(&dev), "cudaGetDevice");
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if ((int)g_dev.size() <= dev) g_dev.resize(dev + 1);
    DevState &d = g_dev[dev];
    if (!d.init) {
        LS_CUDA(cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev), "SM count");
        for (int dt = 0; dt < 4; ++dt) {
            for (int ex = 0; ex < 2; ++ex)
                for (int tm = 0; tm < 2; ++tm) {
                    const Launch L = pick_scan((ls_dtype)dt, ex != 0, tm != 0);
                    LS_CUDA(cudaFuncSetAttribute((const void *)L.fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)L.smem),
                            "cudaFuncSetAttribute(max dynamic smem)");
                    int occ = 0;
                    LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void *)L.fn, L.threads, L.smem),
                            "occupancy query");
                    if (occ < 1) return fail(LS_ERR_CUDA, "scan kernel cannot be resident (smem %zu B)", L.smem);
                    d.occ[dt][ex][tm] = occ;
                }
        }
        const void *rf[4] = {(const void *)&reduce_kernel<uint32_t, kReduceThreads>,
                             (const void *)&reduce_kernel<uint64_t, kReduceThreads>,
                             (const void *)&reduce_kernel<float, kReduceThreads>,
                             (const void *)&reduce_kernel<double, kReduceThreads>};
        for (int dt = 0; dt < 4; ++dt) {
            int occ = 0;
            LS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, rf[dt], kReduceThreads, 0), "occupancy");
            d.reduce_occ[dt] = std::max(occ, 1);
        }
        d.init = true;
    }
    *out = &d;
    return LS_OK;
}

bool valid_dtype(ls_dtype dt) { return dt >= LS_I32 && dt <= LS_F64; }

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

template <typename T>
ls_status launch_carry(const void *totals, int64_t count, int64_t rank, void *carry_out, cudaStream_t s) {
    (void)count;
    carry_kernel<T><<<1, 32, 0, s>>>(static_cast<const T *>(totals), rank, static_cast<T *>(carry_out));
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LS_CUDA(cudaGetLastError(), "carry_kernel launch");
    return LS_OK;
}

ls_status scan_impl(ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in, void *total_out,
                    void *ws, size_t ws_bytes, void *stream, bool excl) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
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
    if (n == 0) {
        if (total_out) {
            if (carry_in) LS_CUDA(cudaMemcpyAsync(total_out, carry_in, es, cudaMemcpyDeviceToDevice, s), "copy carry");
            else LS_CUDA(cudaMemsetAsync(total_out, 0, es, s), "zero total");
        }
        return LS_OK;
    }
    ls_status st = check_ws_header(ws, ws_bytes, ls_workspace_bytes(dt, n));
    if (st != LS_OK) return st;
    DevState *d = nullptr;
    if ((st = device_state(&d)) != LS_OK) return st;

    const bool tma = (((uintptr_t)x | (uintptr_t)y) & 15u) == 0;
    const int64_t M = num_tiles(dt, n, tma);
    const int occ = d->occ[dt][excl][tma];
    const int64_t cap = (int64_t)occ * d->sms;
    const int G = (int)std::min<int64_t>(M, cap);

    const DebugCfg dbg = debug_snapshot();
    ScanParams p;
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
    p.experiment = 0;
    p.delay_red_ns = dbg.delay_red_ns;
    p.delay_scan_ns = dbg.delay_scan_ns;
    // a stalled tile without a watchdog would hang the chain forever
    p.stall_tile = dbg.spin_budget > 0 ? dbg.stall_tile : -1;

    // Cooperative launch: the driver refuses a grid that cannot be fully
    // co-resident, which is the deadlock-freedom precondition of the
    // persistent chain (chainscan/schedsim.py's invariant).
    cudaLaunchConfig_t cfg = {};
    const Launch L = pick_scan(dt, excl, tma);
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3((unsigned)L.threads);
    cfg.dynamicSmemBytes = L.smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    LS_CUDA(cudaLaunchKernelEx(&cfg, L.fn, p), "scan kernel launch");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (dbg.armed()) return read_device_error(ws, s, true);
    return LS_OK;
}

template <typename T>
void launch_reduce(const void *x, int64_t n, void *total_out, void *ws, int grid, cudaStream_t s) {
    reduce_kernel<T, kReduceThreads><<<grid, kReduceThreads, 0, s>>>(static_cast<const T *>(x), n,
                                                                     static_cast<T *>(total_out),
                                                                     static_cast<uint8_t *>(ws));
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
    size_t bytes = kSlotBase + 2 * (size_t)M * sw;
    return (bytes + 255) & ~(size_t)255;
}

ls_status ls_workspace_init(void *ws, size_t ws_bytes, void *stream) {
    if (!ws || ws_bytes < kSlotBase) return fail(LS_ERR_WORKSPACE, "workspace NULL or smaller than its header");
    LS_CUDA(cudaMemsetAsync(ws, 0, ws_bytes, static_cast<cudaStream_t>(stream)), "workspace memset");
    return LS_OK;
}

ls_status ls_inclusive_sum(ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in, void *total_out,
                           void *ws, size_t ws_bytes, void *stream) {
    return scan_impl(dt, x, y, n, carry_in, total_out, ws, ws_bytes, stream, false);
}

ls_status ls_exclusive_sum(ls_dtype dt, const void *x, void *y, int64_t n, const void *carry_in, void *total_out,
                           void *ws, size_t ws_bytes, void *stream) {
    return scan_impl(dt, x, y, n, carry_in, total_out, ws, ws_bytes, stream, true);
}

ls_status ls_reduce_sum(ls_dtype dt, const void *x, int64_t n, void *total_out, void *ws, size_t ws_bytes,
                        void *stream) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (n < 0) return fail(LS_ERR_INVALID_ARG, "n must be >= 0");
    if (!total_out) return fail(LS_ERR_INVALID_ARG, "total_out must be non-NULL");
    const int es = elem_size(dt);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (n == 0) {
        LS_CUDA(cudaMemsetAsync(total_out, 0, es, s), "zero total");
        return LS_OK;
    }
    if (!x || ((uintptr_t)x % es)) return fail(LS_ERR_INVALID_ARG, "x NULL or misaligned");
    ls_status st = check_ws_header(ws, ws_bytes, kSlotBase);
    if (st != LS_OK) return st;
    DevState *d = nullptr;
    if ((st = device_state(&d)) != LS_OK) return st;
    const int64_t per_cta = (int64_t)kReduceThreads * (16 / es) * 4;
    int64_t grid = std::min<int64_t>((n + per_cta - 1) / per_cta, (int64_t)d->reduce_occ[dt] * d->sms);
    grid = std::max<int64_t>(1, std::min<int64_t>(grid, kMaxGrid));
    switch (dt) {
    case LS_I32: launch_reduce<uint32_t>(x, n, total_out, ws, (int)grid, s); break;
    case LS_I64: launch_reduce<uint64_t>(x, n, total_out, ws, (int)grid, s); break;
    case LS_F32: launch_reduce<float>(x, n, total_out, ws, (int)grid, s); break;
    case LS_F64: launch_reduce<double>(x, n, total_out, ws, (int)grid, s); break;
    }
    g_launches.fetch_add(1, std::memory_order_relaxed);
    LS_CUDA(cudaGetLastError(), "reduce kernel launch");
    return LS_OK;
}

ls_status ls_carry_from_totals(ls_dtype dt, const void *totals, int64_t count, int64_t rank, void *carry_out,
                               void *stream) {
    if (!valid_dtype(dt)) return fail(LS_ERR_UNSUPPORTED_DTYPE, "unsupported dtype code %d", (int)dt);
    if (!totals || !carry_out || count < 1 || rank < 0 || rank >= count)
        return fail(LS_ERR_INVALID_ARG, "bad totals/carry_out/count/rank");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    switch (dt) {
    case LS_I32: return launch_carry<uint32_t>(totals, count, rank, carry_out, s);
    case LS_I64: return launch_carry<uint64_t>(totals, count, rank, carry_out, s);
    case LS_F32: return launch_carry<float>(totals, count, rank, carry_out, s);
    case LS_F64: return launch_carry<double>(totals, count, rank, carry_out, s);
    }
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
    const int occ = d->occ[dt][0][1];
    const int64_t M = num_tiles(dt, n, true);
    const Launch L = pick_scan(dt, false, true);
    out[0] = std::min<int64_t>(std::max<int64_t>(M, 1), (int64_t)occ * d->sms);
    out[1] = L.threads;
    out[2] = tile_elems(dt, true);
    out[3] = elem_size(dt) == 4 ? FastCfg<4>::kStages : FastCfg<8>::kStages;
    out[4] = occ;
    out[5] = d->sms;
    return LS_OK;
}

}  // extern "C"
