// Probe: can host-pinned VMM memory (cuMemCreate, location HOST_NUMA) back a gather table on
// this box, and does its 2-MiB mapping granularity change the translation behaviour? (dev aid)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <random>
#include "ut.h"

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)

int main(int argc, char** argv) {
  size_t gib = argc > 1 ? atol(argv[1]) : 16;
  int loc = argc > 2 ? atoi(argv[2]) : 0;  // 0: HOST_NUMA, 1: HOST
  size_t bytes = gib << 30;
  cudaSetDevice(0);
  cudaFree(0);
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = loc == 0 ? CU_MEM_LOCATION_TYPE_HOST_NUMA : CU_MEM_LOCATION_TYPE_HOST;
  prop.location.id = 0;
  size_t gran = 0;
  CK(cuMemGetAllocationGranularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
  printf("granularity %zu\n", gran);
  bytes = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h;
  CK(cuMemCreate(&h, bytes, &prop, 0));
  CUdeviceptr va;
  CK(cuMemAddressReserve(&va, bytes, gran, 0, 0));
  CK(cuMemMap(va, bytes, 0, h, 0));
  CUmemAccessDesc acc[2]{};
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE; acc[0].location.id = 0;
  acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location.type = prop.location.type; acc[1].location.id = 0;
  acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CK(cuMemSetAccess(va, bytes, acc, 2));
  printf("mapped %zu bytes at %p\n", bytes, (void*)va);
  uint8_t* p = (uint8_t*)va;
  for (size_t i = 0; i < bytes; i += 4096) p[i] = (uint8_t)(i >> 12);
  memset(p, 7, 1 << 20);
  printf("cpu write ok\n");
  cudaPointerAttributes at{};
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  printf("attr err=%d type=%d devptr=%p hostptr=%p\n", (int)e, (int)at.type, at.devicePointer, at.hostPointer);
  const uint64_t rb = 512, rows = bytes / rb;
  ut_table* t = ut_register(p, rows, rb);
  char msg[512];
  if (!t) { ut_last_error(msg, sizeof msg); printf("ut_register failed: %s\n", msg); return 1; }
  printf("plan %s\n", ut_plan_name(t));
  size_t n = argc > 3 ? atol(argv[3]) : (1 << 20);
  std::vector<int64_t> idx(n);
  std::mt19937_64 g(1);
  for (auto& x : idx) x = g() % rows;
  int64_t* didx; uint8_t* dout;
  cudaMalloc(&didx, n * 8); cudaMalloc(&dout, n * rb);
  cudaMemcpy(didx, idx.data(), n * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* modes[] = {"reorder=off", "reorder=on"};
  for (int m = 0; m < 2; ++m) {
    ut_set_plan(t, modes[m]);
    for (int r = 0; r < 3; ++r) {
      cudaEventRecord(a); int rc = ut_gather(t, didx, n, dout, 0); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (r == 2) printf("%s rc=%d n=%zu gbs=%.2f\n", modes[m], rc, n, n * rb / ms / 1e6);
    }
  }
  std::vector<uint8_t> chk(rb);
  cudaMemcpy(chk.data(), dout + 5 * rb, rb, cudaMemcpyDeviceToHost);
  printf("check %s\n", memcmp(chk.data(), p + idx[5] * rb, rb) == 0 ? "ok" : "MISMATCH");
  ut_release(t);
  return 0;
}
