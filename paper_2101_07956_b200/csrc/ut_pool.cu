// ut_pool.cu — the unified allocator with block recycling.
//
// PAPER.md §4.4: "A new memory allocator is implemented to govern the memory allocation
// for all unified tensors. It adapts the allocation recycling mechanism from the PyTorch CUDA
// allocator to reduce the number of CUDA API invocations." A freed block is kept, not handed back
// to cudaHostAlloc / cudaMallocManaged, and the next request of the same rounded size takes it:
// the page-locking (pinned) or mapping + cudaMemAdvise (managed) of a new allocation is paid once
// per block instead of once per tensor. Parameters follow DESIGN.md reading R19:
// 512-B rounding, whole-block reuse by exact rounded size, most recently freed first, a byte limit
// that empties the cache before it fails. The backend allocations are also what ut_create uses.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>
#include <new>
#include <unordered_map>
#include <vector>

#include "ut.h"
#include "ut_internal.h"

namespace utx {

int backend_alloc(int kind, int dev, uint64_t bytes, void** out) {
  void* p = nullptr;
  cudaError_t e;
  switch (kind) {
    case UT_ALLOC_PINNED:
      if ((e = cudaHostAlloc(&p, bytes, cudaHostAllocPortable | cudaHostAllocMapped)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(UT_ENOMEM, "cudaHostAlloc(%llu): %s", (unsigned long long)bytes,
                       cudaGetErrorString(e));
      }
      break;
    case UT_ALLOC_MANAGED: {
      int managed = 0;
      cudaDeviceGetAttribute(&managed, cudaDevAttrManagedMemory, dev);
      if (!managed) return set_err(UT_ENOTSUP, "device %d has no managed memory", dev);
      if ((e = cudaMallocManaged(&p, bytes, cudaMemAttachGlobal)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(UT_ENOMEM, "cudaMallocManaged(%llu): %s", (unsigned long long)bytes,
                       cudaGetErrorString(e));
      }
      // the paper's advice for unified tensors (Table 2): pages stay in host memory,
      // the device maps them
      cudaMemLocation cpu{};
      cpu.type = cudaMemLocationTypeHost;
      cpu.id = 0;
      cudaMemLocation gpu{};
      gpu.type = cudaMemLocationTypeDevice;
      gpu.id = dev;
      if ((e = cudaMemAdvise(p, bytes, cudaMemAdviseSetPreferredLocation, cpu)) != cudaSuccess ||
          (e = cudaMemAdvise(p, bytes, cudaMemAdviseSetAccessedBy, gpu)) != cudaSuccess) {
        cudaFree(p);
        return cuda_err(e, "cudaMemAdvise");
      }
      break;
    }
    case UT_ALLOC_SYSTEM:
      if (!(p = malloc(bytes))) return set_err(UT_ENOMEM, "malloc(%llu)", (unsigned long long)bytes);
      break;
    default:
      return set_err(UT_EINVAL, "allocation kind %d has no pool backend", kind);
  }
  *out = p;
  return UT_OK;
}

void backend_free(int kind, void* p) {
  if (kind == UT_ALLOC_PINNED) cudaFreeHost(p);
  else if (kind == UT_ALLOC_MANAGED) cudaFree(p);
  else if (kind == UT_ALLOC_SYSTEM) free(p);
}

}  // namespace utx

using utx::set_err;

struct ut_pool {
  int kind = 0;
  int device = 0;
  uint64_t limit = 0;                                        // 0 = none
  std::mutex mu;
  std::unordered_map<uint64_t, std::vector<void*>> cached;  // capacity -> blocks, last freed last
  std::unordered_map<void*, uint64_t> live;                  // block -> capacity
  uint64_t held = 0;                                         // backend bytes: live + cached
  uint64_t bytes_live = 0, bytes_cached = 0, blocks_cached = 0;
  uint64_t backend_calls = 0, backend_frees = 0, recycled_hits = 0;
};

namespace {

constexpr uint64_t kGranule = 512;

void release_cached_locked(ut_pool* p) {
  for (auto& kv : p->cached) {
    for (void* b : kv.second) utx::backend_free(p->kind, b);
    p->backend_frees += kv.second.size();
    p->held -= kv.first * kv.second.size();
  }
  p->cached.clear();
  p->bytes_cached = 0;
  p->blocks_cached = 0;
}

}  // namespace

namespace utx {

int pool_take(ut_pool* p, uint64_t bytes, void** out, uint64_t* cap_out) {
  if (!p || !out) return set_err(UT_EINVAL, "pool or out pointer is NULL");
  if (bytes > UINT64_MAX - (kGranule - 1)) return set_err(UT_EINVAL, "size %llu overflows", (unsigned long long)bytes);
  const uint64_t cap = (bytes + kGranule - 1) / kGranule * kGranule;
  if (cap_out) *cap_out = cap;
  *out = nullptr;
  if (cap == 0) return UT_OK;                       // the zero-capacity sentinel
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->cached.find(cap);
  if (it != p->cached.end() && !it->second.empty()) {   // recycled: no CUDA call
    void* b = it->second.back();
    it->second.pop_back();
    p->live.emplace(b, cap);
    p->bytes_cached -= cap;
    p->blocks_cached -= 1;
    p->bytes_live += cap;
    p->recycled_hits += 1;
    *out = b;
    return UT_OK;
  }
  if (p->limit && cap > p->limit - p->held) {       // R19: empty the cache, then retry once
    release_cached_locked(p);
    if (cap > p->limit - p->held)
      return set_err(UT_ENOMEM, "pool limit %llu B: %llu B held, %llu B requested",
                     (unsigned long long)p->limit, (unsigned long long)p->held,
                     (unsigned long long)cap);
  }
  int prev = 0;
  if (p->kind != UT_ALLOC_SYSTEM) {
    cudaGetDevice(&prev);
    if (prev != p->device) cudaSetDevice(p->device);
  }
  void* b = nullptr;
  int rc = backend_alloc(p->kind, p->device, cap, &b);
  if (rc == UT_ENOMEM && p->blocks_cached) {        // the backend itself is out: same order
    release_cached_locked(p);
    rc = backend_alloc(p->kind, p->device, cap, &b);
  }
  if (p->kind != UT_ALLOC_SYSTEM && prev != p->device) cudaSetDevice(prev);
  if (rc != UT_OK) return rc;
  p->live.emplace(b, cap);
  p->held += cap;
  p->bytes_live += cap;
  p->backend_calls += 1;
  *out = b;
  return UT_OK;
}

int pool_give(ut_pool* p, void* b) {
  if (!p) return set_err(UT_EINVAL, "pool is NULL");
  if (!b) return UT_OK;                             // the sentinel
  std::lock_guard<std::mutex> lk(p->mu);
  auto it = p->live.find(b);
  if (it == p->live.end()) return set_err(UT_EINVAL, "%p is not a live block of this pool", b);
  const uint64_t cap = it->second;
  p->live.erase(it);
  p->cached[cap].push_back(b);
  p->bytes_live -= cap;
  p->bytes_cached += cap;
  p->blocks_cached += 1;
  return UT_OK;
}

int pool_kind(const ut_pool* p) { return p->kind; }
int pool_device(const ut_pool* p) { return p->device; }

}  // namespace utx

extern "C" {

ut_pool* ut_pool_create(int kind, uint64_t limit_bytes) {
  if (kind != UT_ALLOC_PINNED && kind != UT_ALLOC_MANAGED && kind != UT_ALLOC_SYSTEM)
    return set_err(UT_EINVAL, "allocation kind %d has no pool backend", kind), nullptr;
  int dev = 0;
  if (kind != UT_ALLOC_SYSTEM) {
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return utx::cuda_err(e, "cudaGetDevice"), nullptr;
  }
  ut_pool* p = new (std::nothrow) ut_pool;
  if (!p) return set_err(UT_ENOMEM, "out of host memory"), nullptr;
  p->kind = kind;
  p->device = dev;
  p->limit = limit_bytes;
  return p;
}

int ut_pool_alloc(ut_pool* p, uint64_t bytes, void** host_out, uint64_t* capacity_out) {
  return utx::pool_take(p, bytes, host_out, capacity_out);
}

int ut_pool_free(ut_pool* p, void* host) { return utx::pool_give(p, host); }

int ut_pool_release_cached(ut_pool* p) {
  if (!p) return set_err(UT_EINVAL, "pool is NULL");
  std::lock_guard<std::mutex> lk(p->mu);
  release_cached_locked(p);
  return UT_OK;
}

int ut_pool_get_stats(const ut_pool* cp, ut_pool_stats* st) {
  if (!cp || !st) return set_err(UT_EINVAL, "pool or stats is NULL");
  ut_pool* p = const_cast<ut_pool*>(cp);
  std::lock_guard<std::mutex> lk(p->mu);
  st->backend_calls = p->backend_calls;
  st->backend_frees = p->backend_frees;
  st->recycled_hits = p->recycled_hits;
  st->bytes_live = p->bytes_live;
  st->bytes_cached = p->bytes_cached;
  st->blocks_live = p->live.size();
  st->blocks_cached = p->blocks_cached;
  st->limit_bytes = p->limit;
  return UT_OK;
}

int ut_pool_destroy(ut_pool* p) {
  if (!p) return UT_OK;
  {
    std::lock_guard<std::mutex> lk(p->mu);
    if (!p->live.empty())
      return set_err(UT_EINVAL, "%zu blocks of the pool are still live", p->live.size());
    release_cached_locked(p);
  }
  delete p;
  return UT_OK;
}

}  // extern "C"
