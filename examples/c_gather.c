/* examples/c_gather.c — the C ABI used from plain C (no Python, no torch): register a host
 * table in place, gather rows into device memory, check them against a memcpy loop, then the
 * host-to-host form and the out-of-range report. Build:
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_gather.c \
 *       -L paper_2101_07956_b200 -lut -L /usr/local/cuda/lib64 -lcudart \
 *       -Wl,-rpath,$PWD/paper_2101_07956_b200 -o build/c_gather */
#include <cuda_runtime_api.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "ut.h"

static int fail(const char* what) {
    char msg[512];
    int code = ut_last_error(msg, sizeof msg);
    fprintf(stderr, "FAIL %s: [%d] %s\n", what, code, msg);
    return 1;
}

int main(void) {
    const uint64_t rows = 100000, rb = 52, n = 30000;
    uint8_t* table = aligned_alloc(4096, (rows * rb + 4095) / 4096 * 4096);
    for (uint64_t i = 0; i < rows * rb; ++i) table[i] = (uint8_t)(i * 2654435761u >> 13);
    int64_t* idx = malloc(n * sizeof(int64_t));
    uint64_t x = 88172645463325252ull;
    for (uint64_t i = 0; i < n; ++i) {
        x ^= x << 13; x ^= x >> 7; x ^= x << 17;
        idx[i] = (int64_t)(x % rows);
    }
    ut_table* t = ut_register(table, rows, rb);
    if (!t) return fail("ut_register");
    printf("plan %s\n", ut_plan_name(t));
    int64_t* idx_d;
    uint8_t* out_d;
    if (cudaMalloc((void**)&idx_d, n * sizeof(int64_t)) || cudaMalloc((void**)&out_d, n * rb)) return 1;
    cudaMemcpy(idx_d, idx, n * sizeof(int64_t), cudaMemcpyHostToDevice);
    if (ut_gather(t, idx_d, n, out_d, NULL) != UT_OK) return fail("ut_gather");
    uint8_t* got = malloc(n * rb);
    uint8_t* want = malloc(n * rb);
    cudaMemcpy(got, out_d, n * rb, cudaMemcpyDeviceToHost);
    for (uint64_t i = 0; i < n; ++i) memcpy(want + i * rb, table + (uint64_t)idx[i] * rb, rb);
    if (memcmp(got, want, n * rb)) { fprintf(stderr, "FAIL ut_gather bytes\n"); return 1; }
    memset(got, 0, n * rb);
    if (ut_gather_host(t, idx, n, got, NULL) != UT_OK) return fail("ut_gather_host");
    if (memcmp(got, want, n * rb)) { fprintf(stderr, "FAIL ut_gather_host bytes\n"); return 1; }
    idx[7] = -1;
    cudaMemcpy(idx_d, idx, n * sizeof(int64_t), cudaMemcpyHostToDevice);
    ut_gather(t, idx_d, n, out_d, NULL);
    int64_t bad = 0;
    if (ut_error_pos(t, NULL, &bad) != UT_ERANGE || bad != 7) { fprintf(stderr, "FAIL error_pos %lld\n", (long long)bad); return 1; }
    if (ut_release(t) != UT_OK) return fail("ut_release");
    cudaFree(idx_d);
    cudaFree(out_d);
    printf("C-ABI OK\n");
    return 0;
}
