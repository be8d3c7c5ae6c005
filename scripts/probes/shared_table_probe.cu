// Probe (dev aid, round 2): which host-table memory kinds read random rows at link speed when the
// table is far beyond the GPU's translation reach (papers-shaped, 57 GB), and which of them can be
// SHARED by several processes (one copy per box)? Round 1 measured registered/pinned/VMM host
// memory translation-bound (29 GB/s random 512-B rows over 16 GiB) and managed memory not (51),
// but managed memory is process-private. Candidates added here: system-allocated (HMM) memory
// read directly by GPU threads, private anonymous and MAP_SHARED memfd, with the paper's advice
// (SetPreferredLocation = CPU, SetAccessedBy = GPU) applied through
// cudaMemAdvise on the system allocation.
//
// usage: shared_table_probe MODE GIB [n_rows rb]
//   MODE: managed | register | hmm_anon | hmm_anon_noadv | hmm_memfd | hmm_memfd_noadv |
//         register_memfd
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/mman.h>
#include <unistd.h>
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      printf("{\"error\": \"%s: %s\"}\n", #x, cudaGetErrorString(e_));                 \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

template <int U>
__global__ void gather512(const uint8_t* __restrict__ table, const int64_t* __restrict__ idx,
                          uint64_t n, uint64_t rb, uint8_t* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t warps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t chunks = rb >> 4;
  for (uint64_t r0 = warp * U; r0 < n; r0 += warps * U) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t r = r0 + u;
      if (r < n && lane < chunks) {
        const uint4* src = (const uint4*)(table + (uint64_t)idx[r] * rb) + lane;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(src));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t r = r0 + u;
      if (r < n && lane < chunks) ((uint4*)(out + r * rb))[lane] = v[u];
    }
  }
}

static double now() {
  return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

static cudaError_t advise(void* p, size_t bytes, int dev) {
  cudaMemLocation cpu{};
  cpu.type = cudaMemLocationTypeHost;
  cpu.id = 0;
  cudaMemLocation gpu{};
  gpu.type = cudaMemLocationTypeDevice;
  gpu.id = dev;
  cudaError_t e = cudaMemAdvise(p, bytes, cudaMemAdviseSetPreferredLocation, cpu);
  if (e != cudaSuccess) return e;
  return cudaMemAdvise(p, bytes, cudaMemAdviseSetAccessedBy, gpu);
}

int main(int argc, char** argv) {
  if (argc < 3) {
    printf("usage: %s MODE GIB [n rb]\n", argv[0]);
    return 2;
  }
  const std::string mode = argv[1];
  const double gib = atof(argv[2]);
  const uint64_t n = argc > 3 ? strtoull(argv[3], 0, 10) : (1ull << 20);
  const uint64_t rb = argc > 4 ? strtoull(argv[4], 0, 10) : 512;
  const uint64_t bytes = (uint64_t)(gib * (1ull << 30)) / rb * rb;
  const uint64_t rows = bytes / rb;
  CK(cudaSetDevice(0));
  CK(cudaFree(0));
  int attr[8] = {};
  cudaDeviceGetAttribute(&attr[0], cudaDevAttrPageableMemoryAccess, 0);
  cudaDeviceGetAttribute(&attr[1], cudaDevAttrPageableMemoryAccessUsesHostPageTables, 0);
  cudaDeviceGetAttribute(&attr[2], cudaDevAttrConcurrentManagedAccess, 0);
  cudaDeviceGetAttribute(&attr[3], cudaDevAttrHostRegisterSupported, 0);
  cudaDeviceGetAttribute(&attr[4], cudaDevAttrDirectManagedMemAccessFromHost, 0);
  cudaDeviceGetAttribute(&attr[5], cudaDevAttrHostNativeAtomicSupported, 0);
  printf("{\"attrs\": {\"pageableMemoryAccess\": %d, \"usesHostPageTables\": %d, "
         "\"concurrentManagedAccess\": %d, \"hostRegisterSupported\": %d, "
         "\"directManagedMemAccessFromHost\": %d, \"hostNativeAtomic\": %d}}\n",
         attr[0], attr[1], attr[2], attr[3], attr[4], attr[5]);
  fflush(stdout);

  uint8_t* table = nullptr;
  double t0 = now();
  if (mode == "managed") {
    CK(cudaMallocManaged(&table, bytes));
    CK(advise(table, bytes, 0));
  } else if (mode == "register" || mode == "hmm_anon" || mode == "hmm_anon_noadv") {
    table = (uint8_t*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (table == MAP_FAILED) { printf("{\"error\": \"mmap\"}\n"); return 1; }
    madvise(table, bytes, MADV_HUGEPAGE);
  } else if (mode == "hmm_memfd" || mode == "hmm_memfd_noadv" || mode == "register_memfd") {
    int fd = memfd_create("ut_table", 0);
    if (fd < 0 || ftruncate(fd, bytes) != 0) { printf("{\"error\": \"memfd\"}\n"); return 1; }
    table = (uint8_t*)mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    if (table == MAP_FAILED) { printf("{\"error\": \"mmap memfd\"}\n"); return 1; }
    madvise(table, bytes, MADV_HUGEPAGE);
  } else {
    printf("{\"error\": \"unknown mode\"}\n");
    return 2;
  }
  // fill: row r's first 8 bytes = r, the rest a pattern (all pages touched on the CPU)
  for (uint64_t r = 0; r < rows; ++r) {
    uint64_t* w = (uint64_t*)(table + r * rb);
    w[0] = r;
    for (uint64_t k = 1; k < rb / 8; ++k) w[k] = r * 0x9E3779B97F4A7C15ull + k;
  }
  const double fill_s = now() - t0;
  t0 = now();
  if (mode == "register" || mode == "register_memfd") {
    CK(cudaHostRegister(table, bytes, cudaHostRegisterPortable | cudaHostRegisterMapped | cudaHostRegisterReadOnly));
  } else if (mode == "hmm_anon" || mode == "hmm_memfd") {
    cudaError_t e = advise(table, bytes, 0);
    if (e != cudaSuccess) printf("{\"warn\": \"advise: %s\"}\n", cudaGetErrorString(e));
    cudaGetLastError();
  }
  const double setup_s = now() - t0;

  std::vector<int64_t> idx(n);
  std::mt19937_64 g(12345);
  for (auto& x : idx) x = (int64_t)(g() % rows);
  std::vector<int64_t> sorted = idx;
  std::sort(sorted.begin(), sorted.end());
  int64_t *didx, *dsorted;
  uint8_t* dout;
  CK(cudaMalloc(&didx, n * 8));
  CK(cudaMalloc(&dsorted, n * 8));
  CK(cudaMalloc(&dout, n * rb));
  CK(cudaMemcpy(didx, idx.data(), n * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dsorted, sorted.data(), n * 8, cudaMemcpyHostToDevice));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const int64_t* ix) -> float {
    cudaEventRecord(a);
    gather512<4><<<sms * 2, 256>>>(table, ix, n, rb, dout);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
  };
  // first touch over the whole table (ordered), which for HMM/managed may fault mappings in
  std::vector<int64_t> all;
  t0 = now();
  float first = run(didx);
  const double first_wall = now() - t0;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) { printf("{\"error\": \"kernel: %s\"}\n", cudaGetErrorString(e)); return 1; }
  std::vector<float> rnd, ord;
  for (int i = 0; i < 6; ++i) rnd.push_back(run(didx));
  for (int i = 0; i < 4; ++i) ord.push_back(run(dsorted));
  // another random list (new pages) to see if first-touch cost persists
  for (auto& x : idx) x = (int64_t)(g() % rows);
  CK(cudaMemcpy(didx, idx.data(), n * 8, cudaMemcpyHostToDevice));
  float fresh = run(didx);
  float fresh2 = run(didx);
  // parity spot check
  std::vector<uint64_t> chk(n);
  CK(cudaMemcpy2D(chk.data(), 8, dout, rb, 8, n, cudaMemcpyDeviceToHost));
  uint64_t bad = 0;
  for (uint64_t i = 0; i < n; ++i) bad += chk[i] != (uint64_t)idx[i];
  std::sort(rnd.begin(), rnd.end());
  std::sort(ord.begin(), ord.end());
  const double mb = n * rb / 1e6;
  // where do the pages live after the run? (HMM may have migrated them)
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  printf("{\"mode\": \"%s\", \"table_gib\": %.2f, \"rows\": %llu, \"rb\": %llu, \"n\": %llu, "
         "\"fill_s\": %.1f, \"setup_s\": %.2f, \"first_ms\": %.2f, \"first_wall_s\": %.2f, "
         "\"first_gbs\": %.2f, \"random_gbs_median\": %.2f, \"random_gbs_best\": %.2f, "
         "\"sorted_gbs_median\": %.2f, \"fresh_list_gbs\": %.2f, \"fresh_list_again_gbs\": %.2f, "
         "\"bad_rows\": %llu, \"gpu_used_gib\": %.2f}\n",
         mode.c_str(), bytes / double(1ull << 30), (unsigned long long)rows, (unsigned long long)rb,
         (unsigned long long)n, fill_s, setup_s, first, first_wall, mb / first, mb / rnd[rnd.size() / 2],
         mb / rnd[0], mb / ord[ord.size() / 2], mb / fresh, mb / fresh2, (unsigned long long)bad,
         (total_b - free_b) / double(1ull << 30));
  return 0;
}
