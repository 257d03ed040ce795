/* c_abi_demo.c — the C ABI (include/lscan.h) used from plain C, no torch:
 * allocate with the CUDA runtime, scan i32 / f64 inclusive + exclusive on the
 * device, check against a host fold, and run the host-buffer entry.
 *
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_abi_demo.c \
 *       -L paper_1604_04815_b200/_lib -llscan -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_1604_04815_b200/_lib -o c_abi_demo && ./c_abi_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "lscan.h"

#define CK(call)                                                                              \
    do {                                                                                      \
        ls_status s_ = (call);                                                                \
        if (s_ != LS_OK) {                                                                    \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, ls_status_string(s_), ls_last_error_detail()); \
            return 1;                                                                         \
        }                                                                                     \
    } while (0)

static uint64_t rng = 88172645463325252ull;
static uint64_t next(void) { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return rng; }

int main(void) {
    const int64_t n = 10 * 1000 * 1000 + 7;
    int32_t *hx = malloc(n * sizeof(int32_t)), *hy = malloc(n * sizeof(int32_t));
    double *fx = malloc(n * sizeof(double)), *fy = malloc(n * sizeof(double));
    for (int64_t i = 0; i < n; ++i) {
        hx[i] = (int32_t)next();
        fx[i] = ((double)(next() >> 11) / 9007199254740992.0) * 2.0 - 1.0;
    }
    void *dx, *dy, *ws;
    size_t wsb = ls_workspace_bytes(LS_F64, n);  /* >= the i32 need */
    if (cudaMalloc(&dx, n * 8) || cudaMalloc(&dy, n * 8) || cudaMalloc(&ws, wsb)) return 1;
    CK(ls_workspace_init(ws, wsb, NULL));

    /* i32 inclusive, wrapping: bit-exact against a host fold */
    cudaMemcpy(dx, hx, n * 4, cudaMemcpyHostToDevice);
    CK(ls_inclusive_sum(LS_I32, dx, dy, n, NULL, NULL, ws, wsb, NULL));
    cudaMemcpy(hy, dy, n * 4, cudaMemcpyDeviceToHost);
    uint32_t acc = 0;
    int64_t bad = 0;
    for (int64_t i = 0; i < n; ++i) { acc += (uint32_t)hx[i]; bad += (uint32_t)hy[i] != acc; }
    printf("i32 inclusive: %lld mismatches\n", (long long)bad);
    if (bad) return 2;

    /* i32 exclusive max */
    CK(ls_exclusive_scan(LS_OP_MAX, LS_I32, dx, dy, n, NULL, NULL, ws, wsb, NULL));
    cudaMemcpy(hy, dy, n * 4, cudaMemcpyDeviceToHost);
    int32_t m = INT32_MIN;
    for (int64_t i = 0; i < n; ++i) { bad += hy[i] != m; if (hx[i] > m) m = hx[i]; }
    printf("i32 exclusive max: %lld mismatches\n", (long long)bad);
    if (bad) return 3;

    /* f64 inclusive within the reference envelope 1e-12 * cumsum|x| */
    cudaMemcpy(dx, fx, n * 8, cudaMemcpyHostToDevice);
    CK(ls_inclusive_sum(LS_F64, dx, dy, n, NULL, NULL, ws, wsb, NULL));
    cudaMemcpy(fy, dy, n * 8, cudaMemcpyDeviceToHost);
    double s = 0, env = 0;
    for (int64_t i = 0; i < n; ++i) {
        s += fx[i];
        env += fabs(fx[i]);
        bad += fabs(fy[i] - s) > 1e-12 * env;
    }
    printf("f64 inclusive: %lld outside the envelope\n", (long long)bad);
    if (bad) return 4;

    /* the host-buffer entry (what chained_scan does with numpy arrays), in place */
    memcpy(hy, hx, n * 4);
    CK(ls_scan_host(LS_OP_ADD, LS_I32, hy, hy, n, 0, -1));
    acc = 0;
    for (int64_t i = 0; i < n; ++i) { acc += (uint32_t)hx[i]; bad += (uint32_t)hy[i] != acc; }
    printf("host entry, in place: %lld mismatches\n", (long long)bad);
    if (bad) return 5;
    printf("c_abi_demo ok (%lld launches)\n", (long long)ls_launch_count());
    cudaFree(dx); cudaFree(dy); cudaFree(ws);
    free(hx); free(hy); free(fx); free(fy);
    return 0;
}
