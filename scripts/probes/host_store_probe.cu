// Probe (round 2): do TMA bulk stores (cp.async.bulk.global.shared::cta) into mapped host memory
// travel as larger PCIe writes than SM 16-B stores? ut_gather_host's host->host path is bound by
// the upstream direction: 128-B posted writes carry a 16-B header (x1.125). ncu
// reads pcie__write_bytes of each kernel; this prints the times.
//   k_st16   : every thread stores 16 B, consecutive addresses (what the gather kernels do)
//   k_tma    : each block stages CH bytes in shared memory and writes them with one bulk copy
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

__global__ void k_st16(uint4* __restrict__ dst, uint64_t n16) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (uint64_t)gridDim.x * blockDim.x)
    dst[i] = make_uint4((uint32_t)i, 1u, 2u, 3u);
}

template <int CH>
__global__ void k_tma(uint8_t* __restrict__ dst, uint64_t bytes) {
  __shared__ __align__(128) uint4 buf[CH / 16];
  const uint64_t chunks = bytes / CH;
  for (uint64_t c = blockIdx.x; c < chunks; c += gridDim.x) {
    for (int j = threadIdx.x; j < CH / 16; j += blockDim.x) buf[j] = make_uint4((uint32_t)(c * CH + j), 1u, 2u, 3u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const uint32_t s = (uint32_t)__cvta_generic_to_shared(buf);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(dst + c * CH), "r"(s), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
  const uint64_t bytes = 256ull << 20;
  uint8_t* h = nullptr;
  if (cudaHostAlloc(&h, bytes, cudaHostAllocMapped) != cudaSuccess) return 1;
  uint8_t* d = nullptr;
  cudaHostGetDevicePointer((void**)&d, h, 0);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto report = [&](const char* name) {
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaError_t e = cudaGetLastError();
    printf("{\"probe\": \"host_store\", \"kernel\": \"%s\", \"bytes\": %llu, \"ms\": %.3f, \"gbs\": %.2f, \"err\": \"%s\"}\n",
           name, (unsigned long long)bytes, ms, bytes / (ms / 1e3) / 1e9, cudaGetErrorString(e));
  };
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a);
    k_st16<<<sms * 8, 256>>>((uint4*)d, bytes / 16);
    cudaEventRecord(b);
    report("st16");
    cudaEventRecord(a);
    k_tma<4096><<<sms * 4, 128>>>(d, bytes);
    cudaEventRecord(b);
    report("tma_bulk_4KiB");
    cudaEventRecord(a);
    k_tma<1024><<<sms * 8, 128>>>(d, bytes);
    cudaEventRecord(b);
    report("tma_bulk_1KiB");
  }
  // check the TMA output
  uint64_t bad = 0;
  for (uint64_t c = 0; c < bytes / 1024; c += 997) {
    const uint32_t* w = (const uint32_t*)(h + c * 1024);
    if (w[0] != (uint32_t)(c * 1024) || w[1] != 1u) ++bad;
  }
  printf("{\"check_bad_chunks\": %llu}\n", (unsigned long long)bad);
  return 0;
}
