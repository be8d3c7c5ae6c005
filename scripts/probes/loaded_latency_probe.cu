// Probe (round 2): is the SM-read request ceiling of this host link a fixed number of requests
// in flight (PCIe read tags)? Little's law: requests in flight = request rate x latency. A
// one-thread pointer chase through the host table (each hop one dependent 8-B read of a random
// 128-B line, ld.global.cv) measures the latency a request sees while a load kernel (k_req:
// one random line per warp request, P bytes of it, U requests in flight per warp, B blocks)
// keeps the link busy; the load kernel's own rate comes from CUDA events. If the product
// rate x loaded latency flattens at one value as the load grows, whatever the payload, the
// ceiling is an outstanding-request limit, and that value is its size.
//
// usage: loaded_latency_probe [table_gib]   (managed table, SetPreferredLocation = CPU)
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x)                                                                      \
  do {                                                                             \
    cudaError_t e_ = (x);                                                          \
    if (e_ != cudaSuccess) {                                                       \
      printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(e_));             \
      exit(1);                                                                     \
    }                                                                              \
  } while (0)

__device__ __forceinline__ uint64_t gtime() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread: `hops` dependent reads; line l holds the index of the next line in its first 8 B.
// With `go`, it starts when the load kernel's first block has started.
template <bool CV>
__global__ void k_chase(const uint8_t* table, uint64_t line, int hops, const volatile int* go,
                        unsigned long long* out) {
  if (threadIdx.x != 0) return;
  if (go) {
    const uint64_t ts = gtime();
    while (*go == 0)
      if (gtime() - ts > 2000000000ull) break;   // never spin past 2 s
  }
  const uint64_t t0 = gtime();
  for (int i = 0; i < hops; ++i) {
    uint64_t nxt;
    if (CV)
      asm volatile("ld.global.cv.u64 %0, [%1];" : "=l"(nxt) : "l"(table + (line << 7)) : "memory");
    else
      asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(nxt) : "l"(table + (line << 7)) : "memory");
    line = nxt;
  }
  const uint64_t t1 = gtime();
  out[0] = t1 - t0;
  out[1] = line;
}

template <int U>
__global__ void __launch_bounds__(256) k_load(const uint8_t* __restrict__ table, const uint64_t* __restrict__ lines,
                                              uint64_t n, int P, volatile int* go, uint4* __restrict__ sink) {
  if (go && blockIdx.x == 0 && threadIdx.x == 0) {
    *go = 1;
    __threadfence_system();
  }
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const int lanes = P / 16;
  uint4 acc = make_uint4(0, 0, 0, 0);
  for (uint64_t r0 = warp * U; r0 < n; r0 += nw * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = make_uint4(0, 0, 0, 0);
      const uint64_t r = r0 + u;
      if (r >= n) continue;
      const uint64_t line = __ldg(lines + r);      // every lane: the U index loads batch up
      if (lane < lanes) {
        const uint8_t* p = table + (line << 7) + 16 * lane;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w) : "l"(p));
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
  if ((acc.x & 0xFFFFF) == 0x12345) sink[0] = acc;
}

// Sequential 16-B stores into mapped host memory (the write half of a host->host gather).
__global__ void k_store(uint4* __restrict__ a, uint64_t n16, const volatile int* go) {
  if (go) {
    const uint64_t ts = gtime();
    while (*go == 0)
      if (gtime() - ts > 2000000000ull) break;
  }
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16; i += (uint64_t)gridDim.x * blockDim.x)
    a[i] = make_uint4((uint32_t)i, 1, 2, 3);
}

int main(int argc, char** argv) {
  const double gib = argc > 1 ? atof(argv[1]) : 4.0;
  const int only_load = argc > 3 ? atoi(argv[3]) : 0;   // 1: the load kernel alone (no chase)
  const int skip = argc > 4 ? atoi(argv[4]) : 0;        // bit 0: no ring writes, bit 1: no unloaded chase
  const int duplex = argc > 5 ? atoi(argv[5]) : 0;      // 1: only the read load beside host stores
  const uint64_t bytes = (uint64_t)(gib * (1ull << 30)) & ~4095ull;
  CK(cudaSetDevice(0));
  uint8_t* table = nullptr;
  CK(cudaMallocManaged(&table, bytes));
  cudaMemLocation cpu{};
  cpu.type = cudaMemLocationTypeHost;
  cudaMemLocation gpu{};
  gpu.type = cudaMemLocationTypeDevice;
  gpu.id = 0;
  CK(cudaMemAdvise(table, bytes, cudaMemAdviseSetPreferredLocation, cpu));
  CK(cudaMemAdvise(table, bytes, cudaMemAdviseSetAccessedBy, gpu));
  for (uint64_t i = 0; i < bytes; i += 4096) table[i] = 1;   // populate every page on the host
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t n = 1ull << (argc > 2 ? atoi(argv[2]) : 24);   // load requests per launch
  uint64_t* dl;
  uint4* sink;
  int* go;
  unsigned long long* res;
  CK(cudaMalloc(&dl, n * 8));
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&go, 4));
  CK(cudaMallocHost(&res, 16));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::mt19937_64 g(11);
  const int hops = 4000;
  for (uint64_t win : {(uint64_t)(16ull << 20), bytes}) {
    const uint64_t wl = win / 128;
    // the chase ring: 65536 distinct random lines of the window in one random cycle
    const uint64_t ring = std::min<uint64_t>(65536, wl / 2);
    std::vector<uint64_t> ids(ring);
    {
      std::vector<uint8_t> used(wl, 0);
      for (uint64_t j = 0; j < ring;) {
        const uint64_t l = g() % wl;
        if (!used[l]) {
          used[l] = 1;
          ids[j++] = l;
        }
      }
    }
    if (!(skip & 1))
      for (uint64_t j = 0; j < ring; ++j) *(uint64_t*)(table + (ids[j] << 7)) = ids[(j + 1) % ring];
    std::vector<uint64_t> lines(n);
    for (auto& x : lines) x = g() % wl;
    CK(cudaMemcpy(dl, lines.data(), n * 8, cudaMemcpyHostToDevice));
    // unloaded latency
    if (!(skip & 2)) {
    k_chase<true><<<1, 32, 0, s1>>>(table, ids[0], 200, nullptr, res);   // warm the path
    CK(cudaStreamSynchronize(s1));
    k_chase<true><<<1, 32, 0, s1>>>(table, ids[7], hops, nullptr, res);
    CK(cudaStreamSynchronize(s1));
    printf("{\"probe\": \"loaded_latency\", \"window_mib\": %llu, \"load\": \"none\", \"latency_ns\": %.1f}\n",
           (unsigned long long)(win >> 20), (double)res[0] / hops);
    fflush(stdout);
    }
    if (duplex) {
      // saturated random-line reads (P = 128) with a concurrent store stream into pinned host
      // memory of a chosen width: what the host->host gather's writes do to its reads
      static uint8_t* hw = nullptr;
      const uint64_t wbytes = 1ull << 30;
      if (!hw) CK(cudaHostAlloc(&hw, wbytes, cudaHostAllocMapped));
      uint4* hwd;
      CK(cudaHostGetDevicePointer((void**)&hwd, hw, 0));
      cudaStream_t s3;
      CK(cudaStreamCreateWithFlags(&s3, cudaStreamNonBlocking));
      cudaEvent_t c, d;
      cudaEventCreate(&c);
      cudaEventCreate(&d);
      // warm-up: the GPU's first touch of the window and of the store buffer (slow first
      // mappings on this pool's virtualised boxes) stays out of the measured runs
      k_load<1><<<1184, 256, 0, s2>>>(table, dl, n, 128, nullptr, sink);
      k_store<<<148, 256, 0, s3>>>(hwd, wbytes / 16, nullptr);
      CK(cudaDeviceSynchronize());
      for (int sb : {0, 8, 18, 37, 74, 148, 296}) {
        CK(cudaMemset(go, 0, 4));
        CK(cudaDeviceSynchronize());
        k_chase<true><<<1, 32, 0, s1>>>(table, ids[sb % ring], hops, go, res);
        if (sb) {
          cudaEventRecord(c, s3);
          k_store<<<sb, 256, 0, s3>>>(hwd, wbytes / 16, go);
          cudaEventRecord(d, s3);
        }
        cudaEventRecord(a, s2);
        k_load<1><<<1184, 256, 0, s2>>>(table, dl, n, 128, go, sink);
        cudaEventRecord(b, s2);
        CK(cudaDeviceSynchronize());
        float ms = 0, wms = 0;
        cudaEventElapsedTime(&ms, a, b);
        if (sb) cudaEventElapsedTime(&wms, c, d);
        const double rate = n / (ms / 1e3);
        const double lat = (double)res[0] / hops;
        printf("{\"probe\": \"duplex\", \"window_mib\": %llu, \"store_blocks\": %d, \"read_ms\": %.3f, "
               "\"read_requests_per_s_M\": %.1f, \"read_gbs\": %.2f, \"store_ms\": %.3f, \"store_gbs\": %.2f, "
               "\"latency_ns\": %.1f, \"in_flight_little\": %.0f}\n",
               (unsigned long long)(win >> 20), sb, ms, rate / 1e6, rate * 128 / 1e9, wms,
               sb ? wbytes / (wms / 1e3) / 1e9 : 0.0, lat, rate * lat * 1e-9);
        fflush(stdout);
      }
      continue;
    }
    // chase: 0 = none (the load alone), 1 = ld.global.cv, 2 = ld.global.nc
    for (int chase : {0, 1, 2})
    if (!only_load || chase == 0)
    for (int P : {64, 128})
      for (int blocks : {18, 37, 74, 148, 296, 592, 1184})
        for (int U : {1, 4}) {
          if (blocks < 148 && U == 4) continue;
          if (chase != 1 && !only_load && !(P == 128 && ((blocks == 148 && U == 1) || (blocks == 1184 && U == 4)))) continue;
          CK(cudaMemset(go, 0, 4));
          CK(cudaDeviceSynchronize());
          res[0] = 0;
          if (chase == 1)
            k_chase<true><<<1, 32, 0, s1>>>(table, ids[(blocks * 31 + U * 7 + P) % ring], hops, go, res);
          else if (chase == 2)
            k_chase<false><<<1, 32, 0, s1>>>(table, ids[(blocks * 31 + U * 7 + P) % ring], hops, go, res);
          cudaEventRecord(a, s2);
          switch (U) {
            case 1: k_load<1><<<blocks, 256, 0, s2>>>(table, dl, n, P, chase ? go : nullptr, sink); break;
            default: k_load<4><<<blocks, 256, 0, s2>>>(table, dl, n, P, chase ? go : nullptr, sink); break;
          }
          cudaEventRecord(b, s2);
          CK(cudaDeviceSynchronize());
          float ms = 0;
          cudaEventElapsedTime(&ms, a, b);
          const double rate = n / (ms / 1e3);            // load requests / s
          const double lat = (double)res[0] / hops;      // ns per chase hop under that load
          printf("{\"probe\": \"loaded_latency\", \"chase\": \"%s\", \"window_mib\": %llu, \"payload_bytes\": %d, "
                 "\"blocks\": %d, \"U\": %d, \"warps_x_U\": %d, \"load_ms\": %.3f, "
                 "\"requests_per_s_M\": %.1f, \"payload_gbs\": %.2f, \"latency_ns\": %.1f, "
                 "\"chase_ms\": %.3f, \"in_flight_little\": %.0f}\n",
                 chase == 0 ? "none" : chase == 1 ? "cv" : "nc", (unsigned long long)(win >> 20), P, blocks, U, blocks * 8 * U, ms, rate / 1e6,
                 rate * P / 1e9, lat, res[0] / 1e6, rate * lat * 1e-9);
          fflush(stdout);
        }
  }
  return 0;
}
