// Probe: sysmem load latency over the host link (pointer chase through a pinned, mapped host
// buffer) and HBM for comparison; plus throughput vs loads in flight (dev aid).
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>

__global__ void chase(const uint64_t* __restrict__ a, uint64_t start, int hops, uint64_t* out, long long* cycles) {
  uint64_t p = start;
  long long t0 = clock64();
  for (int i = 0; i < hops; ++i) p = a[p];
  long long t1 = clock64();
  *out = p;
  *cycles = t1 - t0;
}

// each warp streams 128-B lines with `inflight` independent 16-B loads per lane outstanding
__global__ void stream_read(const uint4* __restrict__ a, uint64_t n16, int inflight, uint64_t* sink) {
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint32_t acc = 0;
  for (uint64_t base = tid; base < n16; base += stride * inflight) {
    uint4 v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < inflight && base + u * stride < n16) v[u] = __ldg(a + base + u * stride);
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u < inflight && base + u * stride < n16) acc ^= v[u].x ^ v[u].w;
  }
  if (acc == 0x12345678u) *sink = acc;
}

int main() {
  const size_t n = 1ull << 27;   // 1 GiB of uint64
  uint64_t* h;
  cudaHostAlloc(&h, n * 8, cudaHostAllocMapped | cudaHostAllocPortable);
  std::vector<uint64_t> perm(n / 64);
  for (size_t i = 0; i < perm.size(); ++i) perm[i] = i;
  std::shuffle(perm.begin(), perm.end(), std::mt19937_64(1));
  // a random cycle over 512-B strided slots
  for (size_t i = 0; i < perm.size(); ++i) h[perm[i] * 64] = perm[(i + 1) % perm.size()] * 64;
  uint64_t* d; cudaMalloc(&d, n * 8);
  cudaMemcpy(d, h, n * 8, cudaMemcpyHostToDevice);
  uint64_t* hd; cudaHostGetDevicePointer((void**)&hd, h, 0);
  uint64_t* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int hops = 4000;
  for (int which = 0; which < 2; ++which) {
    const uint64_t* a = which ? d : hd;
    chase<<<1, 1>>>(a, 0, 100, out, cyc);
    chase<<<1, 1>>>(a, perm[7] * 64, hops, out, cyc);
    long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("{\"probe\": \"pointer_chase\", \"memory\": \"%s\", \"cycles_per_hop\": %.0f, \"ns_per_hop_at_clock_rate\": %.0f}\n",
           which ? "hbm" : "sysmem (pinned, mapped)", (double)c / hops, (double)c / hops / (clk_khz / 1e6));
  }
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int blocks : {8, 16, 37, 74, 148, 296, 592}) {
    for (int inflight : {1, 4}) {
      stream_read<<<blocks, 256>>>((const uint4*)hd, n / 2, inflight, out);
      cudaEventRecord(e0);
      stream_read<<<blocks, 256>>>((const uint4*)hd, n / 2, inflight, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double bytes_in_flight = (double)blocks * 256 * 16 * inflight;
      printf("{\"probe\": \"stream_read_sysmem\", \"blocks\": %d, \"loads_in_flight_per_thread\": %d, \"bytes_in_flight\": %.0f, \"gbs\": %.2f}\n",
             blocks, inflight, bytes_in_flight, n * 8 / ms / 1e6);
    }
  }
  return 0;
}
