// Probe: can the copy engine gather rows? cudaMemcpyBatchAsync of n per-row H2D copies (the
// paper's rejected "one cudaMemcpy per row", with CUDA 12.8's batch API) vs the SM
// gather (dev aid).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

int main() {
  const size_t rows = 2449029, rb = 400;
  uint8_t* table;
  cudaHostAlloc(&table, rows * rb, cudaHostAllocMapped | cudaHostAllocPortable);
  for (size_t i = 0; i < rows * rb; i += 4096) table[i] = 1;
  for (size_t n : {1000, 10000, 100000, 462000}) {
    std::vector<void*> src(n), dst(n);
    std::vector<size_t> sz(n, rb);
    uint8_t* out;
    cudaMalloc(&out, n * rb);
    std::mt19937_64 g(n);
    for (size_t i = 0; i < n; ++i) {
      src[i] = table + (g() % rows) * rb;
      dst[i] = out + i * rb;
    }
    cudaMemcpyAttributes attr{};
    attr.srcAccessOrder = cudaMemcpySrcAccessOrderStream;
    attr.flags = 0;
    size_t ai = 0, fail = 0;
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaError_t e = cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), n, &attr, &ai, 1, &fail, st);
    cudaStreamSynchronize(st);
    if (e != cudaSuccess) { printf("{\"n\": %zu, \"error\": \"%s\"}\n", n, cudaGetErrorString(e)); continue; }
    cudaEventRecord(e0, st);
    e = cudaMemcpyBatchAsync(dst.data(), src.data(), sz.data(), n, &attr, &ai, 1, &fail, st);
    cudaEventRecord(e1, st);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"probe\": \"cudaMemcpyBatchAsync per-row H2D\", \"n\": %zu, \"row_bytes\": %zu, \"ms\": %.3f, \"gbs\": %.3f, \"copies_per_s_M\": %.2f}\n",
           n, rb, ms, n * rb / ms / 1e6, n / ms / 1e3);
    cudaFree(out);
  }
  return 0;
}
