// Probe (round 2, VERDICT r1 task 4): what bounds SM-issued sysmem reads — bytes or requests?
//
// Each warp request reads P bytes (lanes 0..P/16-1, one 16-B load each) of ONE random 128-B line
// of a host table, U requests in flight per warp, over a grid of B blocks x 256 threads. Sweeps
// P in {16, 32, 64, 96, 128} (one line per request), the bytes in flight (B, U), and two ways a
// 256-B pair of lines might travel as one request: the L2::256B promotion hint on the loads and
// a cp.async.bulk.prefetch.L2 of the 256-B pair before the loads. Reports requests/s and payload
// GB/s (CUDA events); ncu's syslts__t_requests_aperture_sysmem_op_read and pcie__read_bytes /
// pcie__write_bytes for the same launches are taken by scripts/gpu_request_probe.sh.
// Calibration kernels: a sequential whole-line read of exactly CAL bytes (pcie__read_bytes per
// payload byte) and a sequential 16-B store stream of CAL bytes into mapped host memory
// (pcie__write_bytes per payload byte).
//
// usage: request_rate_probe [table_gib] [kind: managed|pinned]
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(e_));             \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

enum Mode { PLAIN = 0, PROMOTE256 = 1, PREFETCH256 = 2, PAIR = 3 };

__device__ __forceinline__ uint4 ld16(const uint8_t* p, int mode) {
  uint4 v;
  if (mode == PROMOTE256)
    asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  else
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}

// lines[r] = 128-B line index of request r. P bytes per request; in PAIR / *256 modes a request
// covers the 256-B aligned pair (line & ~1, line | 1): lanes 0..15, 16 B each.
template <int U>
__global__ void __launch_bounds__(256) k_req(const uint8_t* __restrict__ table, const uint64_t* __restrict__ lines,
                                             uint64_t n, int P, int mode, uint4* __restrict__ sink) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const bool pair = mode != PLAIN;
  const int lanes = pair ? 16 : P / 16;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint64_t r0 = warp * U; r0 < n; r0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = make_uint4(0, 0, 0, 0);
      const uint64_t r = r0 + u;
      if (r >= n) continue;
      uint64_t line = __ldg(lines + r);
      const uint8_t* base;
      if (pair) {
        base = table + ((line & ~1ull) << 7);
        if (mode == PREFETCH256 && lane == 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], 256;" ::"l"(base) : "memory");
        if (lane < 16) v[u] = ld16(base + 16 * lane, mode);   // 8 lanes per line, 2 lines
      } else {
        base = table + (line << 7);
        if (lane < lanes) v[u] = ld16(base + 16 * lane, mode);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      acc.x ^= v[u].x;
      acc.y ^= v[u].y;
      acc.z ^= v[u].z;
      acc.w ^= v[u].w;
    }
  }
  (void)lanes;
  if ((acc.x & 0xFFFFF) == 0x12345) sink[0] = acc;
}

// sequential whole-line read of `bytes` (calibration of pcie__read_bytes)
__global__ void k_seq_read(const uint4* __restrict__ a, uint64_t n16, uint4* sink) {
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x) {
    uint4 v = __ldg(a + i);
    acc.x ^= v.x;
    acc.w ^= v.w;
  }
  if (acc.x == 0x9876543u) sink[0] = acc;
}

// sequential 16-B stores of `bytes` into mapped host memory (calibration of pcie__write_bytes)
__global__ void k_seq_write(uint4* __restrict__ a, uint64_t n16) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 4.0;
  const std::string kind = argc > 2 ? argv[2] : "managed";
  const uint64_t bytes = (uint64_t)(gib * (1ull << 30)) & ~255ull;
  const uint64_t nlines = bytes / 128;
  CK(cudaSetDevice(0));
  uint8_t* table = nullptr;
  if (kind == "managed") {
    CK(cudaMallocManaged(&table, bytes));
    cudaMemLocation cpu{};
    cpu.type = cudaMemLocationTypeHost;
    cudaMemLocation gpu{};
    gpu.type = cudaMemLocationTypeDevice;
    gpu.id = 0;
    CK(cudaMemAdvise(table, bytes, cudaMemAdviseSetPreferredLocation, cpu));
    CK(cudaMemAdvise(table, bytes, cudaMemAdviseSetAccessedBy, gpu));
  } else {
    CK(cudaHostAlloc(&table, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
  }
  for (uint64_t i = 0; i < bytes; i += 4096) table[i] = (uint8_t)i;
  const uint64_t n = 1ull << 22;   // requests per launch
  std::vector<uint64_t> lines(n);
  std::mt19937_64 g(7);
  for (auto& x : lines) x = g() % nlines;
  uint64_t* dl;
  uint4* sink;
  CK(cudaMalloc(&dl, n * 8));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMemcpy(dl, lines.data(), n * 8, cudaMemcpyHostToDevice));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto run = [&](int P, int mode, int blocks, int U) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      switch (U) {
        case 1: k_req<1><<<blocks, 256>>>(table, dl, n, P, mode, sink); break;
        case 2: k_req<2><<<blocks, 256>>>(table, dl, n, P, mode, sink); break;
        case 4: k_req<4><<<blocks, 256>>>(table, dl, n, P, mode, sink); break;
        default: k_req<8><<<blocks, 256>>>(table, dl, n, P, mode, sink); break;
      }
      cudaEventRecord(b);
      CK(cudaEventSynchronize(b));
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = std::min(best, ms);
    }
    const char* mn[] = {"plain", "promote256", "prefetch256", "pair"};
    const int lines_per_req = mode == PLAIN ? 1 : 2;
    const double payload = mode == PLAIN ? P : 256;
    const double inflight = (double)blocks * 8 * U * payload;
    printf("{\"probe\": \"request_rate\", \"table\": \"%s\", \"table_gib\": %.1f, \"mode\": \"%s\", "
           "\"payload_bytes\": %.0f, \"lines_per_request\": %d, \"blocks\": %d, \"U\": %d, "
           "\"bytes_in_flight\": %.0f, \"ms\": %.3f, \"warp_requests_per_s_M\": %.1f, "
           "\"line_requests_per_s_M\": %.1f, \"payload_gbs\": %.2f}\n",
           kind.c_str(), gib, mn[mode], payload, lines_per_req, blocks, U, inflight, best,
           n / (best / 1e3) / 1e6, n * lines_per_req / (best / 1e3) / 1e6, n * payload / (best / 1e3) / 1e9);
    fflush(stdout);
  };
  // 1) payload sweep at full occupancy
  for (int P : {16, 32, 64, 96, 128}) run(P, PLAIN, sms * 8, 4);
  // 2) bytes-in-flight sweep at 64 B and 128 B
  for (int P : {64, 128})
    for (int blocks : {37, 74, 148, 296, 592, 1184})
      for (int U : {1, 4})
        run(P, PLAIN, blocks, U);
  // 3) a 256-B pair of lines: plain loads, L2::256B promotion, bulk prefetch to L2 first
  for (int mode : {PAIR, PROMOTE256, PREFETCH256}) run(256, mode, sms * 8, 4);
  // 4) locality: the same random single-line requests confined to a window of the table, and
  //    the full-table list sorted by address (what a reorder stage would give)
  auto label = [&](const char* what) {
    printf("{\"probe\": \"locality\", \"case\": \"%s\"}\n", what);
  };
  for (uint64_t win : {1ull << 24, 1ull << 26, 1ull << 28, 1ull << 30, 1ull << 32}) {
    if (win > bytes) break;
    std::vector<uint64_t> w(n);
    for (uint64_t i = 0; i < n; ++i) w[i] = lines[i] % (win / 128);
    CK(cudaMemcpy(dl, w.data(), n * 8, cudaMemcpyHostToDevice));
    char buf[64];
    snprintf(buf, sizeof buf, "window_%llu_MiB", (unsigned long long)(win >> 20));
    label(buf);
    run(128, PLAIN, sms * 8, 4);
    run(64, PLAIN, sms * 8, 4);
  }
  {
    std::vector<uint64_t> srt = lines;
    std::sort(srt.begin(), srt.end());
    CK(cudaMemcpy(dl, srt.data(), n * 8, cudaMemcpyHostToDevice));
    label("sorted_full_table");
    run(128, PLAIN, sms * 8, 4);
    run(64, PLAIN, sms * 8, 4);
    // sorted, but a request every 4th line only (sparser than 1 line per 4 KiB page)
    for (uint64_t i = 0; i < n; ++i) srt[i] = (i * 37) % nlines;
    std::sort(srt.begin(), srt.end());
    CK(cudaMemcpy(dl, srt.data(), n * 8, cudaMemcpyHostToDevice));
    label("strided_37_lines_sorted");
    run(128, PLAIN, sms * 8, 4);
    CK(cudaMemcpy(dl, lines.data(), n * 8, cudaMemcpyHostToDevice));
  }
  // 5) calibration kernels (ncu reads pcie__read_bytes / pcie__write_bytes of these)
  const uint64_t cal = 256ull << 20;
  uint8_t* hw;
  CK(cudaHostAlloc(&hw, cal, cudaHostAllocMapped));
  cudaEventRecord(a);
  k_seq_read<<<sms * 8, 256>>>((const uint4*)table, cal / 16, sink);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\": \"calibration_seq_read\", \"bytes\": %llu, \"ms\": %.3f, \"gbs\": %.2f}\n",
         (unsigned long long)cal, ms, cal / (ms / 1e3) / 1e9);
  uint4* hwd;
  CK(cudaHostGetDevicePointer((void**)&hwd, hw, 0));
  cudaEventRecord(a);
  k_seq_write<<<sms * 8, 256>>>(hwd, cal / 16);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  cudaEventElapsedTime(&ms, a, b);
  printf("{\"probe\": \"calibration_seq_write\", \"bytes\": %llu, \"ms\": %.3f, \"gbs\": %.2f}\n",
         (unsigned long long)cal, ms, cal / (ms / 1e3) / 1e9);
  return 0;
}
