/* examples/c_box.c — the box form from plain C: ONE library-owned managed table (the paper's
 * to("unified"), ut_create UT_ALLOC_MANAGED) gathered on every visible GPU from ONE host thread
 * with ut_gather_multi, each GPU its own index list on its own stream; every output checked
 * against a memcpy loop. `c_box [gpus [workers]]`: workers > gpus maps several entries onto one
 * device (a test on a one-GPU box). Build as examples/c_gather.c. */
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

int main(int argc, char** argv) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev < 1) { fprintf(stderr, "no GPU\n"); return 1; }
    int gpus = argc > 1 ? atoi(argv[1]) : ndev;
    if (gpus < 1 || gpus > ndev) gpus = ndev;
    int workers = argc > 2 ? atoi(argv[2]) : gpus;
    if (workers < 1 || workers > 64) workers = gpus;
    const uint64_t rows = 200000, rb = 512, n = 50000;
    cudaSetDevice(0);
    void* host = NULL;
    ut_table* t = ut_create(NULL, rows, rb, UT_ALLOC_MANAGED, &host);
    if (!t) return fail("ut_create");
    uint8_t* table = host;
    for (uint64_t i = 0; i < rows * rb; ++i) table[i] = (uint8_t)(i * 2654435761u >> 11);
    int devs[64];
    const int64_t* idx_d[64];
    void* out_d[64];
    uint64_t cnt[64];
    ut_stream_t st[64];
    int64_t* idx[64];
    uint64_t x = 88172645463325252ull;
    for (int k = 0; k < workers; ++k) {
        devs[k] = k % gpus;
        cudaSetDevice(devs[k]);
        cnt[k] = n - 1000 * (uint64_t)k;
        idx[k] = malloc(cnt[k] * sizeof(int64_t));
        for (uint64_t i = 0; i < cnt[k]; ++i) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            idx[k][i] = (int64_t)(x % rows);
        }
        int64_t* d;
        if (cudaMalloc((void**)&d, cnt[k] * sizeof(int64_t)) || cudaMalloc(&out_d[k], cnt[k] * rb)) return 1;
        cudaMemcpy(d, idx[k], cnt[k] * sizeof(int64_t), cudaMemcpyHostToDevice);
        idx_d[k] = d;
        cudaStream_t s;
        cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
        st[k] = (ut_stream_t)s;
    }
    cudaSetDevice(0);
    if (ut_gather_multi(t, workers, devs, idx_d, cnt, out_d, st) != UT_OK) return fail("ut_gather_multi");
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != 0) { fprintf(stderr, "FAIL current device not restored (%d)\n", cur); return 1; }
    for (int k = 0; k < workers; ++k) {
        cudaSetDevice(devs[k]);
        cudaStreamSynchronize((cudaStream_t)st[k]);
        uint8_t* got = malloc(cnt[k] * rb);
        cudaMemcpy(got, out_d[k], cnt[k] * rb, cudaMemcpyDeviceToHost);
        for (uint64_t i = 0; i < cnt[k]; ++i)
            if (memcmp(got + i * rb, table + (uint64_t)idx[k][i] * rb, rb)) {
                fprintf(stderr, "FAIL worker %d row %llu\n", k, (unsigned long long)i);
                return 1;
            }
        free(got);
    }
    cudaSetDevice(0);
    if (ut_release(t) != UT_OK) return fail("ut_release");
    printf("C-BOX OK gpus=%d workers=%d\n", gpus, workers);
    return 0;
}
