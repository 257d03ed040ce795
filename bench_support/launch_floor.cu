// launch_floor.cu — lab (not the product): host cost per launch and device
// latency per dependent launch for the small-n regime, to separate what the
// scan kernels cost from what any launch costs on this box.
//
//   empty <<<1,1024>>>            plain launch
//   empty cluster(1) Ex           cudaLaunchKernelEx + cluster attribute
//   empty cooperative Ex          cudaLaunchKernelEx + cooperative attribute
//   ls_inclusive_scan n=2^10..    the product C ABI (cluster / persistent kernels)
//
// Each is timed (a) host wall per call of 20000 back-to-back calls (host
// bound when the kernel is short), (b) device time per call of 200 calls
// replayed from a captured CUDA graph.  Prints one JSON object.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <string>
#include <vector>

#include "lscan.h"

__global__ void empty_kernel(int *p) {
    if (p && threadIdx.x == 1023 && blockIdx.x == 12345) *p = 1;
}

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
            exit(1);                                                                     \
        }                                                                                \
    } while (0)

static double host_us(cudaStream_t s, const std::function<void()> &f, int reps = 20000) {
    for (int i = 0; i < 100; ++i) f();
    CK(cudaStreamSynchronize(s));
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; ++i) f();
    CK(cudaStreamSynchronize(s));
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / reps;
}

static double graph_us(cudaStream_t s, const std::function<void()> &f, int reps = 200) {
    f();
    CK(cudaStreamSynchronize(s));
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < reps; ++i) f();
    CK(cudaStreamEndCapture(s, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    CK(cudaGraphLaunch(ge, s));
    CK(cudaStreamSynchronize(s));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    float best = 1e30f;
    for (int k = 0; k < 5; ++k) {
        CK(cudaEventRecord(a, s));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        best = ms < best ? ms : best;
    }
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
    return best * 1e3 / reps;
}

int main() {
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    std::string out = "{";
    auto add = [&](const std::string &k, double h, double g) {
        char buf[256];
        snprintf(buf, sizeof buf, "%s\"%s\": {\"host_us\": %.2f, \"graph_us\": %.2f}", out.size() > 1 ? ", " : "",
                 k.c_str(), h, g);
        out += buf;
        fprintf(stderr, "%s host %.2f graph %.2f\n", k.c_str(), h, g);
    };

    auto plain = [&] { empty_kernel<<<1, 1024, 0, s>>>(nullptr); };
    add("empty_plain", host_us(s, plain), graph_us(s, plain));

    auto ex = [&](int kind) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(1);
        cfg.blockDim = dim3(1024);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        if (kind == 1) {
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 1;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
        } else {
            attr[0].id = cudaLaunchAttributeCooperative;
            attr[0].val.cooperative = 1;
        }
        cfg.attrs = attr;
        cfg.numAttrs = kind ? 1 : 0;
        int *np = nullptr;
        CK(cudaLaunchKernelEx(&cfg, empty_kernel, np));
    };
    add("empty_ex_noattr", host_us(s, [&] { ex(0); }), graph_us(s, [&] { ex(0); }));
    add("empty_ex_cluster1", host_us(s, [&] { ex(1); }), graph_us(s, [&] { ex(1); }));
    add("empty_ex_cooperative", host_us(s, [&] { ex(2); }), graph_us(s, [&] { ex(2); }));

    for (int lg : {10, 14, 18, 20}) {
        const int64_t n = 1ll << lg;
        void *x, *y, *ws;
        CK(cudaMalloc(&x, n * 4));
        CK(cudaMalloc(&y, n * 4));
        CK(cudaMemset(x, 1, n * 4));
        const size_t wb = ls_workspace_bytes(LS_I32, n);
        CK(cudaMalloc(&ws, wb));
        ls_workspace_init(ws, wb, s);
        for (int path : {0, 1}) {
            ls_debug_force_path(path);
            auto f = [&] {
                if (ls_inclusive_sum(LS_I32, x, y, n, nullptr, nullptr, ws, wb, s) != LS_OK) {
                    fprintf(stderr, "scan failed: %s\n", ls_last_error_detail());
                    exit(1);
                }
            };
            add(std::string("scan_i32_2^") + std::to_string(lg) + (path ? "_persistent" : "_auto"), host_us(s, f, 5000),
                graph_us(s, f));
        }
        ls_debug_force_path(0);
        CK(cudaFree(x));
        CK(cudaFree(y));
        CK(cudaFree(ws));
    }
    out += "}";
    printf("%s\n", out.c_str());
    return 0;
}
