// ut.cu — registration layer, plan selection and C ABI of the unified-tensor gather.
//
// Implements include/ut.h. The "unified tensor" of PyTorch-Direct is host memory that GPU
// threads dereference directly; here the caller's table is pinned
// and mapped in place (cudaHostRegister Portable|Mapped[|ReadOnly]) instead of copied into a new
// allocation (reading R1), and `unified_tensor[gpu_tensor]`
// is ut_gather. The kernels are in ut_kernels.cuh.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <unordered_map>
#include <vector>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unistd.h>

#include "ut.h"
#include "ut_internal.h"
#include "ut_kernels.cuh"
#include "ut_scan.cuh"

namespace utx {

thread_local int g_err_code = UT_OK;
thread_local char g_err_msg[512] = "";

int set_err(int code, const char* fmt, ...) {
  g_err_code = code;
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err_msg, sizeof g_err_msg, fmt, ap);
  va_end(ap);
  return code;
}

int cuda_err(cudaError_t e, const char* what) {
  return set_err(UT_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// Page-locked and mapped for the GPU (cudaHostAlloc / cudaHostRegister / adopted)? When it is,
// *end receives the end of the allocation range containing `a` if the driver reports it, else 0.
static bool pinned_at(uint64_t a, uint64_t* end) {
  cudaPointerAttributes at{};
  const bool ok = cudaPointerGetAttributes(&at, (const void*)a) == cudaSuccess &&
                  at.type == cudaMemoryTypeHost && at.devicePointer != nullptr;
  cudaGetLastError();
  *end = 0;
  if (!ok) return false;
  using PAttr = CUresult (*)(void*, CUpointer_attribute, CUdeviceptr);
  static const PAttr attr_f = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    if (cudaGetDriverEntryPoint("cuPointerGetAttribute", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return (PAttr) nullptr;
    return reinterpret_cast<PAttr>(fn);
  }();
  CUdeviceptr start = 0;
  size_t size = 0;
  if (attr_f && attr_f(&start, CU_POINTER_ATTRIBUTE_RANGE_START_ADDR, (CUdeviceptr)a) == CUDA_SUCCESS &&
      attr_f(&size, CU_POINTER_ATTRIBUTE_RANGE_SIZE, (CUdeviceptr)a) == CUDA_SUCCESS && size > 0 &&
      (uint64_t)start <= a && a < (uint64_t)start + size)
    *end = (uint64_t)start + size;
  return true;
}

// Make [p, p+bytes) GPU-addressable in place. The common case registers the page-aligned range
// in one call. If part of it is already page-locked (cudaHostAlloc'd by the caller, or pages a
// neighbouring registration holds), the range is walked allocation by allocation: pinned
// stretches are adopted (their extent from the driver's range attributes, else page by page)
// and every unpinned gap is registered, splitting a gap in halves where the driver refuses it
// because a pinned island lies inside. Every byte is covered before the table is used.
int pin_host(const void* p, uint64_t bytes, bool read_only, Pin* out) {
  *out = Pin{};
  int dev = 0, ro_ok = 0;
  cudaGetDevice(&dev);
  if (read_only) cudaDeviceGetAttribute(&ro_ok, cudaDevAttrHostRegisterReadOnlySupported, dev);
  const uint64_t pg = (uint64_t)sysconf(_SC_PAGESIZE);
  const uint64_t lo = (uint64_t)p / pg * pg;
  const uint64_t hi = ((uint64_t)p + bytes + pg - 1) / pg * pg;
  const unsigned flags = cudaHostRegisterPortable | cudaHostRegisterMapped;
  int ro_all = 1;
  auto reg = [&](uint64_t a, uint64_t len) -> cudaError_t {
    cudaError_t e = cudaErrorUnknown;
    if (ro_ok) {
      e = cudaHostRegister((void*)a, len, flags | cudaHostRegisterReadOnly);
      if (e != cudaSuccess) cudaGetLastError();
    }
    if (e != cudaSuccess) {
      e = cudaHostRegister((void*)a, len, flags);
      if (e != cudaSuccess) cudaGetLastError();
      else ro_all = 0;
    }
    if (e == cudaSuccess) out->regs.emplace_back((const uint8_t*)a, len);
    return e;
  };
  auto fail = [&](cudaError_t e, uint64_t len) {
    unpin_host(out);
    if (e == cudaErrorMemoryAllocation)
      return set_err(UT_ENOMEM, "cudaHostRegister(%llu bytes): %s", (unsigned long long)len,
                     cudaGetErrorString(e));
    return cuda_err(e, "cudaHostRegister");
  };
  uint64_t end0 = 0, end1 = 0;
  if (pinned_at((uint64_t)p, &end0) && end0 >= (uint64_t)p + bytes) {
    out->base = (const uint8_t*)lo;   // one pinned allocation holds every byte: adopt it
    out->len = hi - lo;
    return UT_OK;
  }
  cudaError_t e = reg(lo, hi - lo);
  if (e != cudaSuccess && e != cudaErrorHostMemoryAlreadyRegistered &&
      (pinned_at(lo, &end0) || pinned_at(hi - 1, &end1)))
    e = cudaErrorHostMemoryAlreadyRegistered;   // some driver paths report overlap differently
  if (e != cudaSuccess && e != cudaErrorHostMemoryAlreadyRegistered) return fail(e, hi - lo);
  if (e != cudaSuccess) {
    ro_all = 0;                     // adopted stretches keep their owner's flags
    uint64_t a = lo;
    while (a < hi) {
      uint64_t end = 0;
      if (pinned_at(a, &end)) {     // adopt this allocation's stretch
        a = end > a ? std::min(hi, (end + pg - 1) / pg * pg) : a + pg;
        continue;
      }
      // an unpinned gap starting at a: register [a, hi), halving on refusal
      uint64_t len = hi - a;
      for (;;) {
        e = reg(a, len);
        if (e == cudaSuccess) break;
        if (e == cudaErrorMemoryAllocation || len <= pg) return fail(e, len);
        len = (len / 2 + pg - 1) / pg * pg;
      }
      a += len;
    }
  }
  out->base = (const uint8_t*)lo;
  out->len = hi - lo;
  out->read_only = ro_all;
  return UT_OK;
}

void unpin_host(Pin* pin) {
  for (auto& r : pin->regs) cudaHostUnregister(const_cast<uint8_t*>(r.first));
  cudaGetLastError();
  *pin = Pin{};
}

int pin_device_ptr(const Pin& pin, const void* p, uint64_t* dev) {
  int d = 0, same = 0;
  cudaGetDevice(&d);
  cudaDeviceGetAttribute(&same, cudaDevAttrCanUseHostPointerForRegisteredMem, d);
  if (same) {   // UVA: the host address is the device address of registered memory
    *dev = (uint64_t)p;
    return UT_OK;
  }
  // without UVA the device addresses of separate registrations are not contiguous
  if (pin.regs.size() != 1 || pin.regs[0].first != pin.base || pin.regs[0].second != pin.len)
    return set_err(UT_ENOTSUP, "table is not one registration and the device has no UVA");
  void* dp = nullptr;
  cudaError_t e = cudaHostGetDevicePointer(&dp, const_cast<void*>(p), 0);
  if (e != cudaSuccess) return cuda_err(e, "cudaHostGetDevicePointer");
  *dev = (uint64_t)dp;
  return UT_OK;
}

}  // namespace utx

using namespace utx;

namespace {

constexpr int kMaxDev = 64;

// ---- plans ------------------------------------------------------------------------------------
enum PlanKind { P_AUTO = -1, P_NARROW = 0, P_VEC16 = 1, P_VEC16X = 2, P_REALIGN = 3, P_REALIGNX = 4, P_BULK = 5,
                P_PAPER_NAIVE = 6, P_PAPER_SHIFT = 7, P_TMA4 = 8 };

struct Plan {
  PlanKind kind;
  int g;       // lanes per row (single-pass) or element bytes (narrow)
  bool clip;   // realign: table base or end not 16-B aligned
};

const char* plan_name(const Plan& p) {
  switch (p.kind) {
    case P_NARROW:
      switch (p.g) { case 1: return "narrow1"; case 2: return "narrow2"; case 4: return "narrow4";
                     default: return "narrow8"; }
    case P_VEC16:
      switch (p.g) { case 1: return "vec16.g1"; case 2: return "vec16.g2"; case 4: return "vec16.g4";
                     case 8: return "vec16.g8"; case 16: return "vec16.g16"; default: return "vec16.g32"; }
    case P_VEC16X: return "vec16.g32x";
    case P_REALIGN:
      switch (p.g) { case 1: return "realign.g1"; case 2: return "realign.g2"; case 4: return "realign.g4";
                     case 8: return "realign.g8"; case 16: return "realign.g16"; default: return "realign.g32"; }
    case P_REALIGNX: return "realign.g32x";
    case P_BULK: return "bulk";
    case P_TMA4: return "tma4";
    case P_PAPER_NAIVE: return "paper_naive";
    case P_PAPER_SHIFT: return "paper_shift";
    default: return "invalid";
  }
}

int pow2ceil(uint64_t x) {
  int g = 1;
  while ((uint64_t)g < x) g <<= 1;
  return g;
}

// Largest number of 16-B chunks a row spans over the residues (start mod 16) that
// start = a0 + k*rb can take.
uint64_t max_span16(uint64_t a0, uint64_t rb) {
  uint64_t m = 0;
  for (uint64_t k = 0; k < 16; ++k) {
    uint64_t o = (a0 + k * rb) & 15;
    m = std::max(m, (o + rb + 15) / 16);
  }
  return m;
}

// The automatic choice (DESIGN.md §Plan selection), or the forced kind when it is admissible.
bool choose_plan(uint64_t base, uint64_t rows, uint64_t rb, uint64_t out, PlanKind forced, Plan* p) {
  const bool clip = ((base & 15) != 0) || (((base + rows * rb) & 15) != 0);
  const bool natural = (rb == 1 || rb == 2 || rb == 4 || rb == 8) && (base % rb == 0) && (out % rb == 0);
  const bool aligned = ((base | rb | out) & 15) == 0;
  const uint64_t span = std::max(max_span16(base, rb), max_span16(out, rb));
  PlanKind k = forced;
  if (k == P_AUTO) {
    if (natural) k = P_NARROW;
    else if (aligned) k = rb <= 512 ? P_VEC16 : P_VEC16X;
    else k = span <= 32 ? P_REALIGN : P_REALIGNX;
  }
  switch (k) {
    case P_NARROW:
      if (!natural) return false;
      *p = Plan{k, (int)rb, false};
      return true;
    case P_VEC16:
      if (!aligned || rb > 512) return false;
      *p = Plan{k, pow2ceil(rb / 16), false};
      return true;
    case P_VEC16X:
      if (!aligned) return false;
      *p = Plan{k, 32, false};
      return true;
    case P_REALIGN:
      if (span > 32) return false;
      *p = Plan{k, pow2ceil(span), clip};
      return true;
    case P_REALIGNX:
      *p = Plan{k, 32, clip};
      return true;
    case P_TMA4:
      if (!aligned || rb > (uint64_t)ut::kTma4MaxRow || rows >= (1ull << 31)) return false;
      *p = Plan{k, 32, false};
      return true;
    case P_BULK:
      if (!aligned || rb > (uint64_t)ut::kBulkMaxRow) return false;
      *p = Plan{k, 32, false};
      return true;
    case P_PAPER_NAIVE:
    case P_PAPER_SHIFT:
      if (((base | rb | out) & 3) != 0) return false;
      *p = Plan{k, 1, false};
      return true;
    default:
      return false;
  }
}

PlanKind parse_plan(const char* s, bool* ok) {
  *ok = true;
  if (!s || !strcmp(s, "auto")) return P_AUTO;
  if (!strcmp(s, "narrow")) return P_NARROW;
  if (!strcmp(s, "vec16")) return P_VEC16;
  if (!strcmp(s, "vec16x")) return P_VEC16X;
  if (!strcmp(s, "realign")) return P_REALIGN;
  if (!strcmp(s, "realignx")) return P_REALIGNX;
  if (!strcmp(s, "bulk")) return P_BULK;
  if (!strcmp(s, "tma4")) return P_TMA4;
  if (!strcmp(s, "paper_naive")) return P_PAPER_NAIVE;
  if (!strcmp(s, "paper_shift")) return P_PAPER_SHIFT;
  *ok = false;
  return P_AUTO;
}

struct DevState {
  std::atomic<bool> init{false};       // published after the fields below are set
  uint64_t dev_base = 0;               // device address of the table on this device
  unsigned long long* err = nullptr;   // first out-of-range position, ~0 = none
  int sms = 0;
  cudaMemPool_t pool = nullptr;         // stream-ordered scratch for the reorder stage
  // counters (ut_get_stats)
  std::atomic<uint64_t> gathers{0}, launches{0}, rows{0}, bytes{0}, shared{0};
  std::mutex tmu;                       // timing events
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending, spare;
  uint64_t timed = 0;
  double timed_ms = 0.0;
  // ut_gather_host scratch
  static constexpr int kBuf = 3;
  int64_t* idx_buf[kBuf] = {};
  uint8_t* out_buf[kBuf] = {};
  uint64_t buf_rows = 0;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t gathered[kBuf] = {};
  cudaEvent_t drained[kBuf] = {};
  int64_t* idx_all = nullptr;           // ut_gather_host zero-copy path: device copy of idx
  uint64_t idx_cap = 0;
  std::mutex hmu;                       // ut_gather_host: this device's host-form scratch
  CUtensorMap tmap;                     // "tma4" plan: the table as a rows x (rb/4) word tensor
  std::mutex tmap_mu;                   // builds tmap once (never t->mu: ut_gather_host's
  std::atomic<bool> tmap_ok{false};     // caller may hold other locks)
};

}  // namespace

struct ut_table {
  const uint8_t* host = nullptr;
  uint64_t rows = 0, rb = 0, bytes = 0;
  Pin pin;                              // ut_register: pages pinned or adopted in place
  int registered = 0, read_only = 0, device = 0;
  int alloc_kind = -1;                  // ut_create: ut_alloc_kind; -1 = caller memory
  bool direct_va = false;               // device address == host address (managed / VMM)
  ut_pool* pool = nullptr;              // ut_pool_table: ut_release hands the block back
  unsigned long long vmm_handle = 0;    // CUmemGenericAllocationHandle
  uint64_t vmm_bytes = 0;
  PlanKind forced = P_AUTO;
  int reorder = -1;                     // -1 auto, 0 off, 1 on (ut_set_plan "reorder=...")
  bool timing = false;                  // ut_set_plan "timing=on"
  int conc = -1;                        // launch shape: -1 auto, 0 dense, 1 sparse ("conc=...")
  int runs = -1;                        // run merge: -1 auto, 0 off, 1 on ("runs=...")
  int stage = -1;                       // host-output tile staging: -1 auto (= off), 0 off, 1 on ("stage=...")
  int share = -1;                       // neighbour line sharing: -1 auto, 0 off, 1 on ("share=...")
  int exact = -1;                       // reorder: exact row order inside each bucket ("exact=...")
  std::mutex mu;
  DevState dev[kMaxDev];
};

namespace {

// The paper's advice for a unified tensor (Table 2) on one more device: the
// pages stay in host memory (SetPreferredLocation = CPU, set at creation) and `dev` maps them.
int managed_accessed_by(const void* p, uint64_t bytes, int dev) {
  cudaMemLocation gpu{};
  gpu.type = cudaMemLocationTypeDevice;
  gpu.id = dev;
  cudaError_t e = cudaMemAdvise(p, bytes, cudaMemAdviseSetAccessedBy, gpu);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return cuda_err(e, "cudaMemAdvise(SetAccessedBy)");
  }
  return UT_OK;
}

// Per-device resources every table of the process shares, so that a table costs no CUDA
// allocation of its own (§6e: recycled unified tensors are tables too): one stream-ordered scratch
// pool (reorder / share / int32 staging; trimmed when the device's last table is released) and a
// slab of device error words handed out and taken back by the tables.
struct DevShared {
  std::mutex mu;
  cudaStream_t stream = nullptr;        // private, non-blocking: clears a word and waits for it
  cudaMemPool_t pool = nullptr;
  std::vector<unsigned long long*> free_words;
  uint64_t tables = 0;                  // tables holding a word on this device
};
DevShared g_shared[kMaxDev];
constexpr int kWordsPerSlab = 4096;

int shared_take(int dev, cudaMemPool_t* pool, unsigned long long** word) {
  DevShared& d = g_shared[dev];
  std::lock_guard<std::mutex> lk(d.mu);
  cudaError_t e;
  if (!d.stream && (e = cudaStreamCreateWithFlags(&d.stream, cudaStreamNonBlocking)) != cudaSuccess)
    return cuda_err(e, "cudaStreamCreateWithFlags");
  if (!d.pool) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if ((e = cudaMemPoolCreate(&p, &props)) != cudaSuccess) return cuda_err(e, "cudaMemPoolCreate");
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &keep);
    d.pool = p;
  }
  if (d.free_words.empty()) {
    unsigned long long* slab = nullptr;
    if ((e = cudaMalloc(&slab, kWordsPerSlab * sizeof *slab)) != cudaSuccess)
      return cuda_err(e, "cudaMalloc(error words)");
    for (int i = kWordsPerSlab - 1; i >= 0; --i) d.free_words.push_back(slab + i);
  }
  unsigned long long* w = d.free_words.back();
  // complete before the table is handed out: its first gather may run on any stream
  if ((e = cudaMemsetAsync(w, 0xff, sizeof *w, d.stream)) != cudaSuccess ||
      (e = cudaStreamSynchronize(d.stream)) != cudaSuccess)
    return cuda_err(e, "cudaMemsetAsync(error word)");
  d.free_words.pop_back();
  d.tables += 1;
  *pool = d.pool;
  *word = w;
  return UT_OK;
}

void shared_give(int dev, unsigned long long* word) {
  DevShared& d = g_shared[dev];
  std::lock_guard<std::mutex> lk(d.mu);
  d.free_words.push_back(word);
  d.tables -= 1;
  // the last table of the device gone: its scratch goes back (live tables keep theirs warm)
  if (d.pool && d.tables == 0) cudaMemPoolTrimTo(d.pool, 0);
}

// Map a VMM host allocation (cuMemCreate HOST_NUMA) for one more device.
int vmm_grant(const void* va, uint64_t size, int dev) {
  using PAccess = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuMemSetAccess", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return set_err(UT_ENOTSUP, "cuMemSetAccess unavailable");
  CUmemAccessDesc acc{};
  acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc.location.id = dev;
  acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  CUresult r = reinterpret_cast<PAccess>(fn)((CUdeviceptr)va, size, &acc, 1);
  if (r != CUDA_SUCCESS)
    return set_err(UT_ENOTSUP, "cuMemSetAccess(device %d) failed (%d): this VMM host table "
                   "cannot be mapped on that device", dev, (int)r);
  return UT_OK;
}

// Lazily resolve the table's device address and error word on the current device.
int dev_state(const ut_table* ct, DevState** out) {
  ut_table* t = const_cast<ut_table*>(ct);
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
  if (dev < 0 || dev >= kMaxDev) return set_err(UT_ENOTSUP, "device %d beyond %d", dev, kMaxDev);
  DevState* s = &t->dev[dev];
  if (s->init.load(std::memory_order_acquire)) {
    *out = s;
    return UT_OK;
  }
  std::lock_guard<std::mutex> lk(t->mu);
  if (!s->init) {
    uint64_t dev_base = (uint64_t)t->host;
    if (!t->direct_va) {
      if (pin_device_ptr(t->pin, t->host, &dev_base) != UT_OK) return UT_ECUDA;
    }
    if (dev != t->device) {
      // a library-owned table used from another device of the process (one table per box,
      // one thread per GPU): extend the creator's mapping to this device
      int rc = UT_OK;
      if (t->alloc_kind == UT_ALLOC_MANAGED) rc = managed_accessed_by(t->host, t->bytes, dev);
      else if (t->alloc_kind == UT_ALLOC_VMM_HOST) rc = vmm_grant(t->host, t->vmm_bytes, dev);
      if (rc != UT_OK) return rc;
    }
    unsigned long long* err = nullptr;
    cudaMemPool_t pool = nullptr;
    if (int rc = shared_take(dev, &pool, &err)) return rc;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    s->pool = pool;
    s->dev_base = dev_base;
    s->err = err;
    s->sms = sms > 0 ? sms : 148;
    s->init.store(true, std::memory_order_release);
  }
  *out = s;
  return UT_OK;
}

// Resident gather blocks per SM (256 threads each), env override UT_BLOCKS_PER_SM (0 = max).
int blocks_per_sm_cap() {
  static const int cap = [] {
    const char* e = getenv("UT_BLOCKS_PER_SM");
    return (e && *e) ? atoi(e) : -1;
  }();
  return cap;
}

// Resident 256-thread blocks per SM of a kernel, queried once per kernel (the occupancy query
// costs microseconds of host time per call otherwise).
int occupancy(const void* kernel) {
  static std::mutex mu;
  static std::unordered_map<const void*, int> cache;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(kernel);
  if (it != cache.end()) return it->second;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, 256, 0);
  if (per_sm <= 0) per_sm = 1;
  cache[kernel] = per_sm;
  return per_sm;
}

template <typename K>
int grid_for(K kernel, int sms, uint64_t work_warps, int cap_blocks = 0) {
  int per_sm = occupancy((const void*)kernel);
  if (blocks_per_sm_cap() > 0) per_sm = std::min(per_sm, blocks_per_sm_cap());
  else if (blocks_per_sm_cap() < 0 && cap_blocks < 0) per_sm = std::min(per_sm, -cap_blocks);
  uint64_t full = (uint64_t)sms * per_sm;
  static const int max_blocks = [] {
    const char* e = getenv("UT_MAX_BLOCKS");        // A/B knob: cap the gather grid
    return (e && *e) ? atoi(e) : 0;
  }();
  if (max_blocks > 0) full = std::min<uint64_t>(full, (uint64_t)max_blocks);
  if (cap_blocks > 0) full = std::min<uint64_t>(full, (uint64_t)cap_blocks);   // < 0: per SM
  uint64_t need = (work_warps + 7) / 8;
  return (int)std::max<uint64_t>(1, std::min(full, need));
}

#ifndef UT_KU
#define UT_KU 4
#endif
#ifndef UT_KUX
#define UT_KUX 2
#endif
constexpr int kU = UT_KU;    // single-pass: row steps in flight per warp tile
constexpr int kUx = UT_KUX;  // multi-pass: LDG.128 per lane in flight per row iteration
constexpr int kUn = 4;       // narrow: rows per thread in flight

template <typename K>
cudaError_t launch(K kernel, int grid, cudaStream_t st, const ut::GatherArgs& a) {
  kernel<<<grid, 256, 0, st>>>(a);
  return cudaGetLastError();
}

// Launch shape. "dense": every SM full of warps, U row-steps in flight per warp — right while the
// table fits the translation reach. "sparse" (reordered gathers from tables beyond the reach):
// one row-step per warp on 3/8 of the SMs (~440 rows, ~220 KB in flight — enough for the link's
// bandwidth x loaded latency of ~3.7 us), because more rows in flight touch more translation
// pages at once and lose more than they hide (measured sweep: 37 blocks 40.8,
// 55 blocks 43.1, 74 blocks 42.0, 110 blocks 36.9 GB/s on the papers shape).
struct Shape {
  bool sparse;
  int cap_blocks;
};

template <int G, int U, bool PERM>
cudaError_t launch_single_u(const Plan& p, int sms, cudaStream_t st, const ut::GatherArgs& a,
                            int cap) {
  constexpr uint64_t rpt = (32 / G) * U;
  const uint64_t tiles = (a.n + rpt - 1) / rpt;
  if (p.kind == P_VEC16) {
    auto k = ut::k_single<G, U, true, false, PERM>;
    return launch(k, grid_for(k, sms, tiles, cap), st, a);
  }
  if (p.clip) {
    auto k = ut::k_single<G, U, false, true, PERM>;
    return launch(k, grid_for(k, sms, tiles, cap), st, a);
  }
  auto k = ut::k_single<G, U, false, false, PERM>;
  return launch(k, grid_for(k, sms, tiles, cap), st, a);
}

template <int G, bool PERM>
cudaError_t launch_single(const Plan& p, int sms, cudaStream_t st, const ut::GatherArgs& a,
                          const Shape& sh, int cap) {
  if (PERM && sh.sparse) return launch_single_u<G, 1, PERM>(p, sms, st, a, sh.cap_blocks);
  return launch_single_u<G, kU, PERM>(p, sms, st, a, cap);
}

// Dense shape: rows > 128 B are link-bound with 2 resident blocks (16 warps) per SM (products
// 45.3 vs 45.2 GB/s at full occupancy, 256-B rows 49.7 vs 48.3) — the rest of each SM stays
// free for concurrent kernels (the next minibatch's sampler, the training step). Rows <= 128 B
// are request-rate-bound and keep every resident block (128-B rows 29.8 vs 27.7 GB/s).
template <bool PERM>
cudaError_t launch_plan(const Plan& p, int sms, cudaStream_t st, const ut::GatherArgs& a,
                        const Shape& sh) {
  const int cap = sh.sparse ? sh.cap_blocks : (a.rb > 128 ? -2 : 0);
  switch (p.kind) {
    case P_NARROW: {
      const uint64_t warps = (a.n + 32 * kUn - 1) / (32 * kUn);
      switch (p.g) {
        case 1: { auto k = ut::k_narrow<uint8_t, kUn, PERM>; return launch(k, grid_for(k, sms, warps, cap), st, a); }
        case 2: { auto k = ut::k_narrow<uint16_t, kUn, PERM>; return launch(k, grid_for(k, sms, warps, cap), st, a); }
        case 4: { auto k = ut::k_narrow<uint32_t, kUn, PERM>; return launch(k, grid_for(k, sms, warps, cap), st, a); }
        default: { auto k = ut::k_narrow<uint64_t, kUn, PERM>; return launch(k, grid_for(k, sms, warps, cap), st, a); }
      }
    }
    case P_VEC16:
    case P_REALIGN:
      switch (p.g) {
        case 1: return launch_single<1, PERM>(p, sms, st, a, sh, cap);
        case 2: return launch_single<2, PERM>(p, sms, st, a, sh, cap);
        case 4: return launch_single<4, PERM>(p, sms, st, a, sh, cap);
        case 8: return launch_single<8, PERM>(p, sms, st, a, sh, cap);
        case 16: return launch_single<16, PERM>(p, sms, st, a, sh, cap);
        default: return launch_single<32, PERM>(p, sms, st, a, sh, cap);
      }
    case P_VEC16X: {
      auto k = ut::k_multi<kUx, true, false, PERM>;
      return launch(k, grid_for(k, sms, a.n, cap), st, a);
    }
    case P_REALIGNX: {
      if (p.clip) {
        auto k = ut::k_multi<kUx, false, true, PERM>;
        return launch(k, grid_for(k, sms, a.n, cap), st, a);
      }
      auto k = ut::k_multi<kUx, false, false, PERM>;
      return launch(k, grid_for(k, sms, a.n, cap), st, a);
    }
    case P_PAPER_NAIVE:
    case P_PAPER_SHIFT: {
      // the paper's kernels visit rows in index order; with a perm they would not be the paper's
      if (PERM) return cudaErrorInvalidValue;
      const uint64_t threads = a.n * (a.rb >> 2);
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * 8, (threads + 255) / 256));
      if (p.kind == P_PAPER_NAIVE) ut::k_paper<false><<<grid, 256, 0, st>>>(a);
      else ut::k_paper<true><<<grid, 256, 0, st>>>(a);
      return cudaGetLastError();
    }
    case P_TMA4: {
      if (PERM || !a.tmap) return cudaErrorInvalidValue;    // A/B plan: index order only
      constexpr int U = 4;
      const int slot = (int)((4 * a.rb + 127) & ~127ull);
      const int smem = 4 * U * slot;
      cudaFuncSetAttribute(ut::k_tma4<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ut::k_tma4<U>, 128, smem);
      if (per_sm <= 0) per_sm = 1;
      const uint64_t tiles = ((a.n + 3) / 4 + U - 1) / U;
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * per_sm, (tiles + 3) / 4));
      ut::k_tma4<U><<<grid, 128, smem, st>>>(*a.tmap, a);
      return cudaGetLastError();
    }
    case P_BULK: {
      constexpr int U = 4;
      auto k = ut::k_bulk<U, PERM>;
      const int smem = 8 * U * (int)((a.rb + 127) & ~127ull);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      int per_sm = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 256, smem);
      if (per_sm <= 0) per_sm = 1;
      const uint64_t tiles = (a.n + U - 1) / U;
      const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)sms * per_sm, (tiles + 7) / 8));
      k<<<grid, 256, smem, st>>>(a);
      return cudaGetLastError();
    }
    default:
      return cudaErrorInvalidValue;
  }
}

// Translation reorder policy. The GPU's translation of the mapped table
// covers about 1 GiB at full speed (measured: random rows over a 16-GiB table run at 56 vs
// 100 Mrows/s, 2-MiB-bucketed rows at 100); beyond that, visiting the rows grouped by 2-MiB
// region restores link-bound speed. Worth its ~4 small launches only for large gathers.
bool want_reorder(const ut_table* t, uint64_t n);

template <bool PERM>
cudaError_t timed_launch(const ut_table* t, DevState* s, const Plan& p, cudaStream_t st,
                         const ut::GatherArgs& a, bool host_out);
Shape shape_for(const ut_table* t, const DevState* s, bool reordered, uint64_t n, bool host_out);

// Region size of the reorder buckets. Rows > 128 B on tables beyond the translation reach:
// 2-MiB regions (the granularity that restores link speed). Rows <= 128 B, whose
// request rate also gains from visiting neighbouring lines together: 64-KiB regions. Either is
// coarsened until the table has at most ut::kMaxBuckets regions (fewer buckets = fewer atomics).
int bucket_shift(uint64_t table_bytes, uint64_t rb) {
  static const int forced = [] {
    const char* e = getenv("UT_REORDER_SHIFT");     // A/B knob
    return (e && *e) ? atoi(e) : 0;
  }();
  int shift = forced ? forced : (rb > 128 && table_bytes > (1ull << 30)) ? 21 : 16;
  while (((table_bytes - 1) >> shift) + 1 > (uint64_t)ut::kMaxBuckets) ++shift;
  return shift;
}

bool want_runs(const ut_table* t, const Plan& p, uint64_t n);
bool want_exact(const ut_table* t, uint64_t n, uint32_t nb);
template <typename F>
cudaError_t timed(const ut_table* t, DevState* s, cudaStream_t st, F&& fn);

// Host-output tile staging (k_staged, opt-in "stage=on"): for ut_gather_host's direct path, when
// base, rb and out share a 4-B (or wider) alignment and 16 B <= rb <= 8 KiB. Measured no gain:
// whole-line writes leave host->host e2e unchanged at 400-B rows (29.9 vs 29.7 GB/s) and lose at
// 512 B (37.8 vs 39.5) and 2408 B (32.9 vs 34.7) to the tile barriers
// (profiles/r1d/e2e_rb_stage.jsonl), so "auto" keeps per-row stores.
int stage_width(const ut_table* t, uint64_t out) {
  const uint64_t m = (uint64_t)t->host | t->rb | out;
  return (m & 15) == 0 ? 16 : (m & 7) == 0 ? 8 : (m & 3) == 0 ? 4 : 0;
}

bool want_stage(const ut_table* t, uint64_t out, const Plan& p) {
  if (t->stage == 0 || t->rb < 16 || t->rb > 8192 || stage_width(t, out) == 0) return false;
  (void)p;
  return t->stage == 1;
}

cudaError_t launch_staged(const ut_table* t, DevState* s, cudaStream_t st, const ut::GatherArgs& a) {
  const uint32_t tile_rows = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>(ut::kStageMaxRows, ut::kStageBytes / t->rb));
  const uint64_t ntiles = (a.n + tile_rows - 1) / tile_rows;
  auto go = [&](auto k) {
    const int per_sm = occupancy((const void*)k);
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)s->sms * per_sm, ntiles));
    k<<<grid, 256, 0, st>>>(a, tile_rows);
    return cudaGetLastError();
  };
  switch (stage_width(t, a.out)) {
    case 16: return go(ut::k_staged<uint4, 4>);
    case 8: return go(ut::k_staged<uint2, 4>);
    default: return go(ut::k_staged<uint32_t, 4>);
  }
}

int gather_runs(const ut_table* t, DevState* s, const Plan& p, const ut::GatherArgs& a, cudaStream_t st);
bool want_share(const ut_table* t, const Plan& p, uint64_t n, bool dev_n);
int gather_share(const ut_table* t, DevState* s, const ut::GatherArgs& a, cudaStream_t st);

// The table as a 2-D tensor of rows x (rb/4) 32-bit words for the "tma4" plan (built once per
// device; cuTensorMapEncodeTiled through the runtime's driver entry point).
int tensor_map(const ut_table* t, DevState* s) {
  if (s->tmap_ok.load(std::memory_order_acquire)) return UT_OK;
  std::lock_guard<std::mutex> lk(s->tmap_mu);
  if (s->tmap_ok.load(std::memory_order_relaxed)) return UT_OK;
  typedef CUresult (*PEncode)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return set_err(UT_ENOTSUP, "cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {t->rb / 4, t->rows};
  const cuuint64_t strides[1] = {t->rb};
  const cuuint32_t box[2] = {(cuuint32_t)(t->rb / 4), 1};
  const cuuint32_t estr[2] = {1, 1};
  CUresult r = reinterpret_cast<PEncode>(fn)(&s->tmap, CU_TENSOR_MAP_DATA_TYPE_UINT32, 2, (void*)s->dev_base,
                                             dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(UT_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  s->tmap_ok.store(true, std::memory_order_release);
  return UT_OK;
}

int gather_on(const ut_table* t, DevState* s, const int64_t* idx_dev, uint64_t n, void* out_dev,
              cudaStream_t st, bool host_out = false, const uint64_t* n_dev = nullptr,
              uint64_t pos0 = 0) {
  Plan p;
  if (!choose_plan((uint64_t)t->host, t->rows, t->rb, (uint64_t)out_dev, t->forced, &p) &&
      !choose_plan((uint64_t)t->host, t->rows, t->rb, (uint64_t)out_dev, P_AUTO, &p))
    return set_err(UT_EINVAL, "no admissible plan");
  ut::GatherArgs a{s->dev_base, t->rows, t->rb, idx_dev, n, (uint64_t)out_dev, s->err, nullptr, n_dev};
  a.pos0 = pos0;          // this list's offset in the caller's (ut_gather_host's chunks)
  if (p.kind == P_TMA4) {
    int rc = tensor_map(t, s);
    if (rc != UT_OK) return rc;
    a.tmap = &s->tmap;
  }
  cudaError_t e;
  s->rows += n;
  s->bytes += n * t->rb;
  if (want_share(t, p, n, n_dev != nullptr)) {
    const int rc = gather_share(t, s, a, st);
    if (rc != UT_ENOMEM) return rc;          // no room for the slot array: the plain gather below
  }
  const bool runs = want_runs(t, p, n);
  // (the reorder splits gathers into 2^31-row chunks, which a device-side row count cannot follow)
  if (!runs && (!want_reorder(t, n) || p.kind == P_PAPER_NAIVE || p.kind == P_PAPER_SHIFT ||
                p.kind == P_TMA4 || (n_dev && n > (1ull << 31)))) {
    if (host_out && want_stage(t, (uint64_t)out_dev, p)) {
      e = timed(t, s, st, [&] { return launch_staged(t, s, st, a); });
      if (e != cudaSuccess) return cuda_err(e, "staged gather");
      return UT_OK;
    }
    e = timed_launch<false>(t, s, p, st, a, host_out);
    if (e != cudaSuccess) return cuda_err(e, plan_name(p));
    return UT_OK;
  }
  if (runs) return gather_runs(t, s, p, a, st);
  // counting sort of the work items by 2-MiB table region (stream-ordered scratch from the
  // library's pool); n < 2^32 per launch, larger gathers are split.
  const int shift = bucket_shift(t->bytes, t->rb);
  const uint32_t nb = (uint32_t)(((t->bytes - 1) >> shift) + 1);
  const int hsm = (int)(nb * sizeof(uint32_t));
  static const bool smem_ok = [] {
    const int mx = ut::kMaxBuckets * (int)sizeof(uint32_t);
    return cudaFuncSetAttribute(ut::k_bucket_count, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess &&
           cudaFuncSetAttribute(ut::k_bucket_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess &&
           cudaFuncSetAttribute(ut::k_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess;
  }();
  if (!smem_ok) return set_err(UT_ECUDA, "cannot opt in to %d B of shared memory", hsm);
  const uint64_t chunk = 1ull << 31;
  for (uint64_t off = 0; off < n; off += chunk) {
    const uint64_t cnt_n = std::min(chunk, n - off);
    uint32_t* scratch = nullptr;
    const size_t bytes = ((size_t)nb + cnt_n) * sizeof(uint32_t);
    if ((e = cudaMallocFromPoolAsync((void**)&scratch, bytes, s->pool, st)) != cudaSuccess)
      return cuda_err(e, "cudaMallocFromPoolAsync(reorder scratch)");
    uint32_t* cnt = scratch;
    uint32_t* perm = scratch + nb;
    ut::GatherArgs c = a;
    c.idx = idx_dev + off;
    c.n = cnt_n;
    c.pos0 = a.pos0 + off;      // error positions stay positions of the whole list
    c.out = (uint64_t)out_dev + off * t->rb;
    c.perm = perm;
    const uint64_t blocks = std::min<uint64_t>((uint64_t)s->sms * 2, (cnt_n + 2047) / 2048);
    const uint64_t per_block = (cnt_n + blocks - 1) / blocks;
    if ((e = cudaMemsetAsync(cnt, 0, nb * sizeof(uint32_t), st)) != cudaSuccess) {
      cudaFreeAsync(scratch, st);
      return cuda_err(e, "cudaMemsetAsync(buckets)");
    }
    ut::k_bucket_count<<<(int)blocks, 512, hsm, st>>>(c, shift, nb, per_block, cnt);
    ut::k_bucket_scan<<<1, 1024, hsm, st>>>(cnt, nb);
    ut::k_bucket_scatter<<<(int)blocks, 512, hsm, st>>>(c, shift, nb, per_block, cnt, perm);
    s->launches += 3;
    if (want_exact(t, cnt_n, nb)) {     // cnt[] now holds the bucket ends
      ut::k_bucket_sort<<<(int)((nb + 255) / 256), 256, 0, st>>>(c, cnt, nb, perm);
      s->launches += 1;
    }
    e = cudaGetLastError();
    if (e == cudaSuccess) e = timed_launch<true>(t, s, p, st, c, host_out);
    cudaError_t e2 = cudaFreeAsync(scratch, st);
    if (e != cudaSuccess) return cuda_err(e, plan_name(p));
    if (e2 != cudaSuccess) return cuda_err(e2, "cudaFreeAsync(reorder scratch)");
  }
  return UT_OK;
}

// Bracket the gather kernel launched by `fn` with timing events when "timing=on".
template <typename F>
cudaError_t timed(const ut_table* t, DevState* s, cudaStream_t st, F&& fn) {
  std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
  if (t->timing) {
    std::lock_guard<std::mutex> lk(s->tmu);
    if (!s->spare.empty()) {
      ev = s->spare.back();
      s->spare.pop_back();
    } else {
      cudaEventCreate(&ev.first);
      cudaEventCreate(&ev.second);
    }
    cudaEventRecord(ev.first, st);
  }
  cudaError_t e = fn();
  if (e == cudaSuccess) {
    s->gathers += 1;
    s->launches += 1;
  }
  if (t->timing) {
    cudaEventRecord(ev.second, st);
    std::lock_guard<std::mutex> lk(s->tmu);
    s->pending.push_back(ev);
  }
  return e;
}

template <bool PERM>
cudaError_t timed_launch(const ut_table* t, DevState* s, const Plan& p, cudaStream_t st,
                         const ut::GatherArgs& a, bool host_out) {
  return timed(t, s, st, [&] { return launch_plan<PERM>(p, s->sms, st, a, shape_for(t, s, PERM, a.n, host_out)); });
}

Shape shape_for(const ut_table* t, const DevState* s, bool reordered, uint64_t n, bool host_out) {
  static const int env_blocks = [] {
    const char* e = getenv("UT_SPARSE_BLOCKS");     // A/B knob: grid of the sparse shape
    return (e && *e) ? atoi(e) : 0;
  }();
  // sparse when the gather brings few bytes per 2-MiB table region: each region's translation is
  // then amortised over little data, and fewer regions in flight is what keeps the link busy
  const uint64_t regions = std::min<uint64_t>(n, ((t->bytes - 1) >> 21) + 1);
  const bool thin = n * t->rb < (32ull << 10) * regions;
  // stores into mapped host memory add their own latency to every row: keep the dense shape there
  bool sparse = t->conc == 1 ||
                (t->conc == -1 && reordered && !host_out && t->bytes > (1ull << 30) && thin &&
                 t->alloc_kind != UT_ALLOC_MANAGED);
  int cap = env_blocks > 0 ? env_blocks : std::max(1, s->sms * 3 / 8);   // 55 of 148 SMs
  return Shape{sparse, cap};
}

// Run merge: sort the work items exactly by row id and copy each run of
// table-adjacent rows with one warp, so their shared boundary lines are requested once. On the
// products shape (19 % of rows have a selected neighbour, 4 % fewer line requests) the gather
// kernel gains 1.9 % but the sort costs ~0.19 ms per 463K rows, a net loss of 2.6 % — so it is
// opt-in ("runs=on"), never chosen by "auto" (profiles/r1_run_merge.log).
bool want_runs(const ut_table* t, const Plan& p, uint64_t n) {
  if (t->runs != 1 || (p.kind != P_VEC16 && p.kind != P_VEC16X)) return false;
  return n < (1ull << 31);
}

int gather_runs(const ut_table* t, DevState* s, const Plan& p, const ut::GatherArgs& a0, cudaStream_t st) {
  const uint64_t n = a0.n;
  int shift = 12;                                   // buckets of ~64 rows, >= 4 KiB
  while ((1ull << (shift + 1)) <= 64 * t->rb) ++shift;
  while (((t->bytes - 1) >> shift) + 1 > (uint64_t)ut::kMaxBuckets) ++shift;
  const uint32_t nb = (uint32_t)(((t->bytes - 1) >> shift) + 1);
  const uint64_t tiles = n / kScanTile + 2;
  // scratch (uint32 words): cnt[nb], perm[n], flags[n], pos[n], starts[n+1], sums[tiles],
  // then two 8-byte words: the effective n and the run count
  const size_t words = (size_t)nb + 4 * n + 1 + tiles + 6;
  const int hsm = (int)(nb * sizeof(uint32_t));
  static const bool smem_ok = [] {
    const int mx = ut::kMaxBuckets * (int)sizeof(uint32_t);
    return cudaFuncSetAttribute(ut::k_bucket_count, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess &&
           cudaFuncSetAttribute(ut::k_bucket_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess &&
           cudaFuncSetAttribute(ut::k_bucket_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) == cudaSuccess;
  }();
  if (!smem_ok) return set_err(UT_ECUDA, "cannot opt in to %d B of shared memory", hsm);
  uint32_t* scratch = nullptr;
  cudaError_t e;
  if ((e = cudaMallocFromPoolAsync((void**)&scratch, words * sizeof(uint32_t), s->pool, st)) != cudaSuccess)
    return cuda_err(e, "cudaMallocFromPoolAsync(run scratch)");
  uint32_t* cnt = scratch;
  uint32_t* perm = cnt + nb;
  uint32_t* flags = perm + n;
  uint32_t* pos = flags + n;
  uint32_t* starts = pos + n;
  uint32_t* sums = starts + n + 1;
  uint64_t* words64 = (uint64_t*)(((uintptr_t)(sums + tiles) + 7) & ~(uintptr_t)7);
  uint64_t* n_eff = words64;
  uint64_t* n_runs = words64 + 1;
  ut::GatherArgs a = a0;
  a.perm = perm;
  const uint64_t blocks = std::min<uint64_t>((uint64_t)s->sms * 2, (n + 2047) / 2048);
  const uint64_t per_block = (n + blocks - 1) / blocks;
  const int gb = (int)((n + 255) / 256);
  ut::k_eff_n<<<1, 1, 0, st>>>(a0.n_dev, n, n_eff);
  e = cudaMemsetAsync(cnt, 0, nb * sizeof(uint32_t), st);
  if (e != cudaSuccess) {
    cudaFreeAsync(scratch, st);
    return cuda_err(e, "cudaMemsetAsync(run buckets)");
  }
  ut::k_bucket_count<<<(int)blocks, 512, hsm, st>>>(a, shift, nb, per_block, cnt);
  ut::k_bucket_scan<<<1, 1024, hsm, st>>>(cnt, nb);
  ut::k_bucket_scatter<<<(int)blocks, 512, hsm, st>>>(a, shift, nb, per_block, cnt, perm);
  ut::k_bucket_sort<<<(int)((nb + 255) / 256), 256, 0, st>>>(a, cnt, nb, perm);
  ut::k_run_flags<<<gb, 256, 0, st>>>(a, flags);
  scan_u32(flags, pos, n_eff, n, n_runs, sums, st);
  ut::k_run_emit<<<gb, 256, 0, st>>>(a, flags, pos, n_runs, starts);
  s->launches += 7 + (n > (uint64_t)kScanTile ? 3 : 2);
  e = cudaGetLastError();
  if (e == cudaSuccess) {
    e = timed(t, s, st, [&] {
      auto k = ut::k_runs<kUx>;
      ut::k_runs<kUx><<<grid_for(k, s->sms, n, -2), 256, 0, st>>>(a, starts, n_runs);
      return cudaGetLastError();
    });
  }
  cudaError_t e2 = cudaFreeAsync(scratch, st);
  if (e != cudaSuccess) return cuda_err(e, "run-merge gather");
  if (e2 != cudaSuccess) return cuda_err(e2, "cudaFreeAsync(run scratch)");
  return UT_OK;
}

// Neighbour line sharing: vec16 tables with 128 < rb <= 512 whose row boundaries
// are not all on 128-B lines. "auto" takes it for gathers of >= 64K rows that select >= 1/16 of
// the table (so that a selected row's successor is selected often enough to pay for the hash of
// the selection), with the row count known on the host (a device-count gather's max_n is only a
// bound).
bool want_share(const ut_table* t, const Plan& p, uint64_t n, bool dev_n) {
  if (t->share == 0 || p.kind != P_VEC16 || t->rb <= 128 || t->rb > 512) return false;
  if ((((uint64_t)t->host | t->rb) & 127) == 0) return false;     // no partial lines to share
  if (n == 0 || n >= (1ull << 31) || t->rows >= 0xFFFFFFFFull) return false;
  if (t->share == 1) return true;
  if (t->reorder == 1 || t->runs == 1 || dev_n) return false;
  return n >= 65536 && n * 16 >= t->rows;
}

// Scratch: the selection hash, 8 B x 2^bits with 2^bits >= 2n (O(n), not O(rows)), stream-ordered
// from the library's pool. The clear, the mark and the gather are all inside timed(), so
// gather_kernel_ms (and bench's roofline.achieved) carry the whole cost of sharing.
int gather_share(const ut_table* t, DevState* s, const ut::GatherArgs& a, cudaStream_t st) {
  uint32_t bits = 1;
  while ((1ull << bits) < 2 * a.n) ++bits;
  const size_t bytes = (size_t)8 << bits;
  ut::ShareHash hs{nullptr, bits};
  cudaError_t e;
  if ((e = cudaMallocFromPoolAsync((void**)&hs.slots, bytes, s->pool, st)) != cudaSuccess) {
    cudaGetLastError();
    return UT_ENOMEM;
  }
  e = timed(t, s, st, [&] {
    cudaError_t e1 = cudaMemsetAsync(hs.slots, 0, bytes, st);
    if (e1 != cudaSuccess) return e1;
    const int gm = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)s->sms * 8, (a.n + 255) / 256));
    ut::k_share_mark<<<gm, 256, 0, st>>>(a, hs);
    s->launches += 1;
    s->shared += 1;
    const uint64_t tiles = (a.n + kU - 1) / kU;
    if (t->rb > 400) {
      auto k = ut::k_share<kU, true>;
      k<<<grid_for(k, s->sms, tiles, -2), 256, 0, st>>>(a, hs);
    } else {
      auto k = ut::k_share<kU, false>;
      k<<<grid_for(k, s->sms, tiles, -2), 256, 0, st>>>(a, hs);
    }
    return cudaGetLastError();
  });
  cudaError_t e2 = cudaFreeAsync(hs.slots, st);
  if (e != cudaSuccess) return cuda_err(e, "shared-line gather");
  if (e2 != cudaSuccess) return cuda_err(e2, "cudaFreeAsync(share hash)");
  return UT_OK;
}

bool want_reorder(const ut_table* t, uint64_t n) {
  if (t->reorder == 0) return false;
  if (t->reorder == 1) return true;
  // the stage costs ~30 us; it pays from ~64K rows (Fig. 7 replica: 8K-32K rows of 1 KB over a
  // 4-GiB pool lose 5-15 % with it, 128K+ gain), and rows >= 4 KB span enough lines per
  // translation that order does not matter (profiles/r1_fig7_replica*.jsonl)
  if (n < 65536 || t->rb >= 4096) return false;
  // beyond the ~1-GiB translation reach of registered / pinned memory every row size gains;
  // below it — and on managed tables, whose mappings have no such reach limit on this box —
  // only small rows, whose request rate (not bytes) is the limit, gain from visiting
  // neighbouring rows together
  const bool small_rows = t->rb <= 128 && t->bytes > (64ull << 20);
  // managed tables beyond 1 GiB: rows with partial 128-B lines (128 < rb < 1 KiB, rb not a line
  // multiple) are bound by the request rate, which falls with the spread of the requests in
  // flight (translation per new page): 2-MiB bucket order lifts 260-B rows
  // 36.2 -> 40.1 GB/s and 400-B rows 44.0 -> 45.3 on the 16-GiB sweep table; whole-line and
  // >= 1-KiB rows are byte-bound and gain nothing (516 B 45.8 = 45.8, 2052 B 50.0 = 49.9;
  // profiles/r2/r2d/sweep_order.log)
  const bool partial = t->rb > 128 && t->rb < 1024 && (t->rb & 127) != 0;
  if (t->alloc_kind == UT_ALLOC_MANAGED) return small_rows || (partial && t->bytes > (1ull << 30));
  return t->bytes > (1ull << 30) || small_rows;
}

// Exact row order inside each reorder bucket ("exact=on"; k_bucket_sort, one thread per bucket,
// insertion sort of buckets up to 256 items): consecutive work items then touch ascending
// addresses, not just the same 2-MiB region. A/B knob; "auto" decides by measurement
// (DESIGN.md §6).
bool want_exact(const ut_table* t, uint64_t n, uint32_t nb) {
  if (t->exact == 0) return false;
  if (t->exact == 1) return true;
  (void)n;
  (void)nb;
  return false;
}

}  // namespace

extern "C" {

ut_table* ut_register(const void* host_ptr, uint64_t rows, uint64_t row_bytes) {
  if (!host_ptr) return set_err(UT_EINVAL, "host_ptr is NULL"), nullptr;
  if (rows == 0 || row_bytes == 0) return set_err(UT_EINVAL, "rows and row_bytes must be >= 1"), nullptr;
  if (rows > UINT64_MAX / row_bytes) return set_err(UT_EINVAL, "rows*row_bytes overflows"), nullptr;
  const uint64_t bytes = rows * row_bytes;
  if ((uint64_t)host_ptr > UINT64_MAX - bytes) return set_err(UT_EINVAL, "table wraps the address space"), nullptr;

  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice"), nullptr;
  int can_map = 0;
  cudaDeviceGetAttribute(&can_map, cudaDevAttrCanMapHostMemory, dev);
  if (!can_map) return set_err(UT_ENOTSUP, "device %d cannot map host memory", dev), nullptr;

  ut_table* t = new (std::nothrow) ut_table;
  if (!t) return set_err(UT_ENOMEM, "out of host memory"), nullptr;
  t->host = (const uint8_t*)host_ptr;
  t->rows = rows;
  t->rb = row_bytes;
  t->bytes = bytes;
  t->device = dev;

  // Already page-locked and mapped (cudaHostAlloc / a previous registration)? Adopt it;
  // otherwise pin the page-aligned range in place.
  if (pin_host(host_ptr, bytes, true, &t->pin) != UT_OK) {
    delete t;
    return nullptr;
  }
  t->registered = t->pin.registered();
  t->read_only = t->pin.read_only;
  const char* env = getenv("UT_PLAN");
  if (env && *env) {
    bool ok;
    PlanKind k = parse_plan(env, &ok);
    Plan p;
    if (ok && (k == P_AUTO || choose_plan((uint64_t)t->host, rows, row_bytes, 0, k, &p))) t->forced = k;
  }
  const char* renv = getenv("UT_REORDER");
  if (renv && *renv) t->reorder = !strcmp(renv, "on") ? 1 : !strcmp(renv, "off") ? 0 : -1;
  DevState* s;
  if (dev_state(t, &s) != UT_OK) {
    char msg[512];
    int code = ut_last_error(msg, sizeof msg);
    ut_release(t);
    set_err(code, "%s", msg);
    return nullptr;
  }
  g_err_code = UT_OK;
  g_err_msg[0] = 0;
  return t;
}

}  // extern "C"

namespace {

template <typename F>
F driver_fn(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

// cuMemCreate(HOST_NUMA) + reserve + map + access for the device and the host.
int vmm_host_alloc(int dev, uint64_t bytes, void** va_out, uint64_t* size_out,
                   unsigned long long* handle_out) {
  using PGran = CUresult (*)(size_t*, const CUmemAllocationProp*, CUmemAllocationGranularity_flags);
  using PCreate = CUresult (*)(CUmemGenericAllocationHandle*, size_t, const CUmemAllocationProp*,
                               unsigned long long);
  using PReserve = CUresult (*)(CUdeviceptr*, size_t, size_t, CUdeviceptr, unsigned long long);
  using PMap = CUresult (*)(CUdeviceptr, size_t, size_t, CUmemGenericAllocationHandle, unsigned long long);
  using PAccess = CUresult (*)(CUdeviceptr, size_t, const CUmemAccessDesc*, size_t);
  using PRelease = CUresult (*)(CUmemGenericAllocationHandle);
  using PFree = CUresult (*)(CUdeviceptr, size_t);
  auto gran_f = driver_fn<PGran>("cuMemGetAllocationGranularity");
  auto create_f = driver_fn<PCreate>("cuMemCreate");
  auto reserve_f = driver_fn<PReserve>("cuMemAddressReserve");
  auto map_f = driver_fn<PMap>("cuMemMap");
  auto access_f = driver_fn<PAccess>("cuMemSetAccess");
  auto release_f = driver_fn<PRelease>("cuMemRelease");
  auto free_f = driver_fn<PFree>("cuMemAddressFree");
  if (!gran_f || !create_f || !reserve_f || !map_f || !access_f || !release_f || !free_f)
    return set_err(UT_ENOTSUP, "driver VMM entry points unavailable");
  int numa = 0;
  cudaDeviceGetAttribute(&numa, cudaDevAttrHostNumaId, dev);
  CUmemAllocationProp prop{};
  prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  prop.location.type = CU_MEM_LOCATION_TYPE_HOST_NUMA;
  prop.location.id = numa < 0 ? 0 : numa;
  size_t gran = 0;
  if (gran_f(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS || !gran)
    return set_err(UT_ENOTSUP, "cuMemGetAllocationGranularity(HOST_NUMA) failed");
  const uint64_t size = (bytes + gran - 1) / gran * gran;
  CUmemGenericAllocationHandle h = 0;
  if (create_f(&h, size, &prop, 0) != CUDA_SUCCESS)
    return set_err(UT_ENOMEM, "cuMemCreate(HOST_NUMA, %llu bytes) failed", (unsigned long long)size);
  CUdeviceptr va = 0;
  if (reserve_f(&va, size, gran, 0, 0) != CUDA_SUCCESS) {
    release_f(h);
    return set_err(UT_ENOMEM, "cuMemAddressReserve failed");
  }
  CUmemAccessDesc acc[2]{};
  acc[0].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  acc[0].location.id = dev;
  acc[0].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  acc[1].location = prop.location;
  acc[1].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  if (map_f(va, size, 0, h, 0) != CUDA_SUCCESS || access_f(va, size, acc, 2) != CUDA_SUCCESS) {
    free_f(va, size);
    release_f(h);
    return set_err(UT_ECUDA, "cuMemMap/cuMemSetAccess failed");
  }
  *va_out = (void*)va;
  *size_out = size;
  *handle_out = (unsigned long long)h;
  return UT_OK;
}

void vmm_host_free(void* va, uint64_t size, unsigned long long handle) {
  using PUnmap = CUresult (*)(CUdeviceptr, size_t);
  using PRelease = CUresult (*)(CUmemGenericAllocationHandle);
  using PFree = CUresult (*)(CUdeviceptr, size_t);
  auto unmap_f = driver_fn<PUnmap>("cuMemUnmap");
  auto release_f = driver_fn<PRelease>("cuMemRelease");
  auto free_f = driver_fn<PFree>("cuMemAddressFree");
  if (unmap_f) unmap_f((CUdeviceptr)va, size);
  if (release_f) release_f((CUmemGenericAllocationHandle)handle);
  if (free_f) free_f((CUdeviceptr)va, size);
}

}  // namespace

namespace {

// The table of a library-owned allocation p (ut_create, ut_pool_table): record it, set up the
// creating device's state, hand out the host address. On failure the table and p are released.
ut_table* finish_owned(ut_table* t, void* p, uint64_t rows, uint64_t row_bytes, int dev, int kind,
                       ut_pool* pool, void** host_out) {
  t->host = (const uint8_t*)p;
  t->rows = rows;
  t->rb = row_bytes;
  t->bytes = rows * row_bytes;
  t->device = dev;
  t->alloc_kind = kind;
  t->direct_va = kind != UT_ALLOC_PINNED;
  t->pool = pool;
  DevState* s;
  if (dev_state(t, &s) != UT_OK) {
    char msg[512];
    int code = ut_last_error(msg, sizeof msg);
    ut_release(t);
    set_err(code, "%s", msg);
    return nullptr;
  }
  *host_out = p;
  g_err_code = UT_OK;
  g_err_msg[0] = 0;
  return t;
}

}  // namespace

extern "C" {

ut_table* ut_create(const void* src, uint64_t rows, uint64_t row_bytes, int kind, void** host_out) {
  if (!host_out) return set_err(UT_EINVAL, "host_out is NULL"), nullptr;
  if (rows == 0 || row_bytes == 0) return set_err(UT_EINVAL, "rows and row_bytes must be >= 1"), nullptr;
  if (rows > UINT64_MAX / row_bytes) return set_err(UT_EINVAL, "rows*row_bytes overflows"), nullptr;
  const uint64_t bytes = rows * row_bytes;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice"), nullptr;
  void* p = nullptr;
  uint64_t vmm_size = 0;
  unsigned long long vmm_h = 0;
  switch (kind) {
    case UT_ALLOC_PINNED:
    case UT_ALLOC_MANAGED:
      if (utx::backend_alloc(kind, dev, bytes, &p) != UT_OK) return nullptr;
      break;
    case UT_ALLOC_VMM_HOST:
      if (vmm_host_alloc(dev, bytes, &p, &vmm_size, &vmm_h) != UT_OK) return nullptr;
      break;
    default:
      return set_err(UT_EINVAL, "unknown allocation kind %d", kind), nullptr;
  }
  if (src) memcpy(p, src, bytes);
  ut_table* t = new (std::nothrow) ut_table;
  if (!t) {
    if (kind == UT_ALLOC_VMM_HOST) vmm_host_free(p, vmm_size, vmm_h);
    else utx::backend_free(kind, p);
    return set_err(UT_ENOMEM, "out of host memory"), nullptr;
  }
  t->vmm_handle = vmm_h;
  t->vmm_bytes = vmm_size;
  return finish_owned(t, p, rows, row_bytes, dev, kind, nullptr, host_out);
}

ut_table* ut_pool_table(ut_pool* pool, const void* src, uint64_t rows, uint64_t row_bytes,
                        void** host_out) {
  if (!pool || !host_out) return set_err(UT_EINVAL, "pool or host_out is NULL"), nullptr;
  if (rows == 0 || row_bytes == 0) return set_err(UT_EINVAL, "rows and row_bytes must be >= 1"), nullptr;
  if (rows > UINT64_MAX / row_bytes) return set_err(UT_EINVAL, "rows*row_bytes overflows"), nullptr;
  const int kind = utx::pool_kind(pool);
  if (kind != UT_ALLOC_PINNED && kind != UT_ALLOC_MANAGED)
    return set_err(UT_EINVAL, "pool kind %d is not GPU-mapped", kind), nullptr;
  void* p = nullptr;
  if (utx::pool_take(pool, rows * row_bytes, &p, nullptr) != UT_OK) return nullptr;
  if (src) memcpy(p, src, rows * row_bytes);
  ut_table* t = new (std::nothrow) ut_table;
  if (!t) {
    utx::pool_give(pool, p);
    return set_err(UT_ENOMEM, "out of host memory"), nullptr;
  }
  // the block's backend mapping was made on the pool's device; dev_state extends it to others
  return finish_owned(t, p, rows, row_bytes, utx::pool_device(pool), kind, pool, host_out);
}

int ut_gather(const ut_table* t, const int64_t* idx_dev, uint64_t n, void* out_dev, ut_stream_t stream) {
  if (!t) return set_err(UT_EINVAL, "table is NULL");
  if (n == 0) return UT_OK;
  if (!idx_dev || !out_dev) return set_err(UT_EINVAL, "idx_dev/out_dev is NULL");
  if (n > UINT64_MAX / t->rb) return set_err(UT_EINVAL, "n*row_bytes overflows");
  DevState* s;
  int rc = dev_state(t, &s);
  if (rc != UT_OK) return rc;
  return gather_on(t, s, idx_dev, n, out_dev, (cudaStream_t)stream);
}

int ut_gather_i32(const ut_table* t, const int32_t* idx_dev, uint64_t n, void* out_dev, ut_stream_t stream) {
  if (!t) return set_err(UT_EINVAL, "table is NULL");
  if (n == 0) return UT_OK;
  if (!idx_dev || !out_dev) return set_err(UT_EINVAL, "idx_dev/out_dev is NULL");
  if (n > UINT64_MAX / t->rb || n > UINT64_MAX / sizeof(int64_t))
    return set_err(UT_EINVAL, "n*row_bytes overflows");
  DevState* s;
  int rc = dev_state(t, &s);
  if (rc != UT_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  int64_t* wide = nullptr;
  cudaError_t e = cudaMallocFromPoolAsync((void**)&wide, n * sizeof(int64_t), s->pool, st);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(UT_ENOMEM, "index scratch of %llu rows", (unsigned long long)n);
  }
  const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)s->sms * 8, (n + 255) / 256));
  ut::k_widen_i32<<<grid, 256, 0, st>>>(idx_dev, wide, n);
  s->launches += 1;
  rc = (e = cudaGetLastError()) != cudaSuccess ? cuda_err(e, "k_widen_i32")
                                               : gather_on(t, s, wide, n, out_dev, st);
  e = cudaFreeAsync(wide, st);
  if (rc == UT_OK && e != cudaSuccess) rc = cuda_err(e, "cudaFreeAsync(index scratch)");
  return rc;
}

int ut_gather_multi(const ut_table* t, int count, const int* devs, const int64_t* const* idx_dev,
                    const uint64_t* n, void* const* out_dev, const ut_stream_t* streams) {
  if (!t) return set_err(UT_EINVAL, "table is NULL");
  if (count < 1 || !devs || !idx_dev || !n || !out_dev)
    return set_err(UT_EINVAL, "count < 1 or a NULL array");
  int cur = 0;
  cudaError_t e = cudaGetDevice(&cur);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
  int rc = UT_OK;
  for (int k = 0; k < count && rc == UT_OK; ++k) {
    if ((e = cudaSetDevice(devs[k])) != cudaSuccess) {
      rc = cuda_err(e, "cudaSetDevice");
      break;
    }
    rc = ut_gather(t, idx_dev[k], n[k], out_dev[k], streams ? streams[k] : nullptr);
  }
  cudaSetDevice(cur);
  return rc;
}

int ut_gather_dn(const ut_table* t, const int64_t* idx_dev, const uint64_t* n_dev, uint64_t max_n,
                 void* out_dev, ut_stream_t stream) {
  if (!t || !n_dev) return set_err(UT_EINVAL, "table or n_dev is NULL");
  if (max_n == 0) return UT_OK;
  if (!idx_dev || !out_dev) return set_err(UT_EINVAL, "idx_dev/out_dev is NULL");
  if (max_n >= (1ull << 31)) return set_err(UT_EINVAL, "max_n must be < 2^31");
  if (max_n > UINT64_MAX / t->rb) return set_err(UT_EINVAL, "max_n*row_bytes overflows");
  DevState* s;
  int rc = dev_state(t, &s);
  if (rc != UT_OK) return rc;
  return gather_on(t, s, idx_dev, max_n, out_dev, (cudaStream_t)stream, false, n_dev);
}

}  // extern "C"

namespace {
// Is every byte of [a, a+bytes) page-locked and mapped, so that kernel stores through the device
// address of `a` land in it? Walks the range allocation by allocation (the driver's range
// attributes): two adjacent pinned allocations qualify only where the host address is the device
// address (UVA), and an unpinned stretch anywhere in the middle disqualifies the range — the
// caller then refuses it instead of faulting. Where the driver reports no range extent, the first
// and last bytes decide.
// Error exit of ut_gather_host: wait for the copies already enqueued (they read the caller's idx
// and write its output) without replacing the error message the caller is about to return.
void drain_keep_error(cudaStream_t a, cudaStream_t b) {
  cudaStreamSynchronize(a);
  if (b) cudaStreamSynchronize(b);
  cudaGetLastError();
}

bool host_range_mapped(uint64_t a, uint64_t bytes, const void* dev_ptr) {
  const uint64_t hi = a + bytes;
  const bool uva = (uint64_t)dev_ptr == a;
  uint64_t p = a, end = 0;
  while (p < hi) {
    if (!pinned_at(p, &end)) return false;
    if (end == 0) return pinned_at(hi - 1, &end);
    if (end >= hi) return true;
    if (!uva) return false;
    p = end;
  }
  return true;
}
}  // namespace

extern "C" {

int ut_gather_host(const ut_table* ct, const int64_t* idx_host, uint64_t n, void* out_host,
                   ut_stream_t stream) {
  if (!ct) return set_err(UT_EINVAL, "table is NULL");
  if (n == 0) return UT_OK;
  if (!idx_host || !out_host) return set_err(UT_EINVAL, "idx_host/out_host is NULL");
  if (n > UINT64_MAX / ct->rb) return set_err(UT_EINVAL, "n*row_bytes overflows");
  ut_table* t = const_cast<ut_table*>(ct);
  DevState* s;
  int rc = dev_state(t, &s);
  if (rc != UT_OK) return rc;
  // per-device lock of the host-form scratch only: gathers on other devices run concurrently
  std::lock_guard<std::mutex> lk(s->hmu);
  cudaStream_t st = (cudaStream_t)stream;
  cudaError_t e;
  // Fast path: out_host is page-locked and mapped, so the gather kernel stores the rows straight
  // into it over the link (one pass, no HBM round trip, no copy engine); the index list is copied
  // to the device once (8 B/row) so the kernel's reads on the link are table rows only.
  cudaPointerAttributes oa{};
  void* out_mapped = nullptr;
  if (cudaPointerGetAttributes(&oa, out_host) == cudaSuccess && oa.type == cudaMemoryTypeHost &&
      oa.devicePointer != nullptr) {
    if (!host_range_mapped((uint64_t)out_host, n * t->rb, oa.devicePointer)) {
      cudaGetLastError();
      // neither path can take it: kernel stores would fault in the unlocked stretch and the copy
      // engine refuses a destination that is only partly page-locked
      return set_err(UT_EINVAL, "out_host is only partly page-locked (%llu bytes from its first "
                     "pinned byte are not one mapped range): pass wholly pinned or wholly "
                     "pageable memory", (unsigned long long)(n * t->rb));
    }
    out_mapped = oa.devicePointer;
  }
  cudaGetLastError();
  // (measured, round 2, papers-shaped managed table: direct stores 36.7 GB/s host->host vs the
  // copy-engine pipeline's 32.6 at its best chunk size, 23.8-32.0 over 2-64 MiB chunks,
  // profiles/r2/r2h/e2e_variants.log; registered tables: direct 29-31 vs 20)
  if (out_mapped && !getenv("UT_HOST_PIPELINE")) {
    if (s->idx_cap < n) {
      // grown geometrically (x1.5, whole MiB): a reallocation synchronises the device, and
      // minibatch sizes vary by a few percent from step to step
      const uint64_t want = std::max<uint64_t>(n, s->idx_cap + s->idx_cap / 2);
      const uint64_t cap = ((want * sizeof(int64_t) + (1u << 20) - 1) >> 20 << 20) / sizeof(int64_t);
      if (s->idx_all) cudaFree(s->idx_all);
      s->idx_all = nullptr;
      s->idx_cap = 0;
      if (cudaMalloc(&s->idx_all, cap * sizeof(int64_t)) != cudaSuccess) {
        cudaGetLastError();
        return set_err(UT_ENOMEM, "device index scratch of %llu rows", (unsigned long long)cap);
      }
      s->idx_cap = cap;
    }
    if ((e = cudaMemcpyAsync(s->idx_all, idx_host, n * sizeof(int64_t), cudaMemcpyHostToDevice,
                             st)) != cudaSuccess)
      return cuda_err(e, "cudaMemcpyAsync(idx H2D)");
    if ((rc = gather_on(t, s, s->idx_all, n, out_mapped, st, true)) != UT_OK) {
      drain_keep_error(st, nullptr);     // the idx copy may still read idx_host: finish it
      return rc;
    }
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_err(e, "sync stream");
    return UT_OK;
  }
  // Otherwise: chunks of rows gathered into device scratch and copied back by the copy engine
  // on a second stream, so the link's two directions overlap.
  static const uint64_t chunk_bytes = [] {
    const char* e = getenv("UT_HOST_CHUNK");          // A/B knob (bytes of rows per chunk)
    return (e && *e) ? (uint64_t)atoll(e) : (8ull << 20);
  }();
  const uint64_t chunk = std::max<uint64_t>(1, chunk_bytes / t->rb);
  const uint64_t want = std::min<uint64_t>(chunk, n);
  if (s->buf_rows < want) {
    for (int b = 0; b < DevState::kBuf; ++b) {
      cudaFree(s->idx_buf[b]);
      cudaFree(s->out_buf[b]);
      s->idx_buf[b] = nullptr;
      s->out_buf[b] = nullptr;
    }
    s->buf_rows = 0;
    for (int b = 0; b < DevState::kBuf; ++b) {
      if (cudaMalloc(&s->idx_buf[b], want * sizeof(int64_t)) != cudaSuccess ||
          cudaMalloc(&s->out_buf[b], want * t->rb) != cudaSuccess) {
        cudaGetLastError();
        return set_err(UT_ENOMEM, "device scratch of %llu rows", (unsigned long long)want);
      }
    }
    s->buf_rows = want;
  }
  if (!s->copy_stream) {
    if ((e = cudaStreamCreateWithFlags(&s->copy_stream, cudaStreamNonBlocking)) != cudaSuccess)
      return cuda_err(e, "cudaStreamCreate");
    for (int b = 0; b < DevState::kBuf; ++b) {
      cudaEventCreateWithFlags(&s->gathered[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&s->drained[b], cudaEventDisableTiming);
    }
  }
  const uint64_t per = s->buf_rows;
  uint64_t k = 0;
  for (uint64_t off = 0; off < n; off += per, ++k) {
    const int b = (int)(k % DevState::kBuf);
    const uint64_t cnt = std::min(per, n - off);
    if (k >= DevState::kBuf) cudaStreamWaitEvent(st, s->drained[b], 0);
    // on an error after earlier chunks were enqueued, their copies still read idx_host and write
    // out_host: finish them before returning, so the caller may free both
    if ((e = cudaMemcpyAsync(s->idx_buf[b], idx_host + off, cnt * sizeof(int64_t),
                             cudaMemcpyHostToDevice, st)) != cudaSuccess) {
      rc = cuda_err(e, "cudaMemcpyAsync(idx H2D)");
      drain_keep_error(st, s->copy_stream);
      return rc;
    }
    if ((rc = gather_on(t, s, s->idx_buf[b], cnt, s->out_buf[b], st, false, nullptr, off)) != UT_OK) {
      drain_keep_error(st, s->copy_stream);
      return rc;
    }
    cudaEventRecord(s->gathered[b], st);
    cudaStreamWaitEvent(s->copy_stream, s->gathered[b], 0);
    if ((e = cudaMemcpyAsync((uint8_t*)out_host + off * t->rb, s->out_buf[b], cnt * t->rb,
                             cudaMemcpyDeviceToHost, s->copy_stream)) != cudaSuccess) {
      rc = cuda_err(e, "cudaMemcpyAsync(rows D2H)");
      drain_keep_error(st, s->copy_stream);
      return rc;
    }
    cudaEventRecord(s->drained[b], s->copy_stream);
  }
  if ((e = cudaStreamSynchronize(s->copy_stream)) != cudaSuccess) return cuda_err(e, "sync copy stream");
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return cuda_err(e, "sync stream");
  return UT_OK;
}

int ut_release(ut_table* t) {
  if (!t) return UT_OK;
  int rc = UT_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < kMaxDev; ++d) {
    DevState& s = t->dev[d];
    if (!s.init && !s.copy_stream && !s.buf_rows) continue;
    cudaSetDevice(d);
    for (int b = 0; b < DevState::kBuf; ++b) {
      if (s.idx_buf[b]) cudaFree(s.idx_buf[b]);
      if (s.out_buf[b]) cudaFree(s.out_buf[b]);
      if (s.gathered[b]) cudaEventDestroy(s.gathered[b]);
      if (s.drained[b]) cudaEventDestroy(s.drained[b]);
    }
    if (s.copy_stream) cudaStreamDestroy(s.copy_stream);
    if (s.idx_all) cudaFree(s.idx_all);
    for (auto* v : {&s.pending, &s.spare})
      for (auto& ev : *v) {
        cudaEventDestroy(ev.first);
        cudaEventDestroy(ev.second);
      }
    if (s.err) shared_give(d, s.err);   // no gather in flight (contract): the word is free
  }
  cudaSetDevice(cur);
  for (auto& r : t->pin.regs) {
    cudaError_t e = cudaHostUnregister(const_cast<uint8_t*>(r.first));
    if (e != cudaSuccess) rc = cuda_err(e, "cudaHostUnregister");
  }
  if (t->pool) utx::pool_give(t->pool, const_cast<uint8_t*>(t->host));   // cached, not freed
  else if (t->alloc_kind == UT_ALLOC_PINNED || t->alloc_kind == UT_ALLOC_MANAGED)
    utx::backend_free(t->alloc_kind, const_cast<uint8_t*>(t->host));
  else if (t->alloc_kind == UT_ALLOC_VMM_HOST)
    vmm_host_free(const_cast<uint8_t*>(t->host), t->vmm_bytes, t->vmm_handle);
  delete t;
  return rc;
}

int ut_error_pos(const ut_table* t, ut_stream_t stream, int64_t* first_bad) {
  if (!t || !first_bad) return set_err(UT_EINVAL, "NULL argument");
  DevState* s;
  int rc = dev_state(t, &s);
  if (rc != UT_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  unsigned long long v = ~0ull;
  cudaError_t e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(e, "cudaStreamSynchronize");
  e = cudaMemcpy(&v, s->err, sizeof v, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(error word)");
  // cleared on `stream` and waited for: a gather enqueued after this call, on any stream, can
  // not race the clear (cudaMemset on the legacy stream may still be pending at return)
  e = cudaMemsetAsync(s->err, 0xff, sizeof v, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemsetAsync(error word)");
  if (v == ~0ull) {
    *first_bad = -1;
    return UT_OK;
  }
  *first_bad = (int64_t)v;
  return UT_ERANGE;
}

int ut_last_error(char* msg, size_t cap) {
  if (msg && cap) {
    strncpy(msg, g_err_msg, cap - 1);
    msg[cap - 1] = 0;
  }
  return g_err_code;
}

const char* ut_plan_name(const ut_table* t) {
  if (!t) return "invalid";
  Plan p;
  if (!choose_plan((uint64_t)t->host, t->rows, t->rb, 0, t->forced, &p) &&
      !choose_plan((uint64_t)t->host, t->rows, t->rb, 0, P_AUTO, &p))
    return "invalid";
  return plan_name(p);
}

const char* ut_plan_probe(uint64_t base, uint64_t rows, uint64_t row_bytes, uint64_t out) {
  if (rows == 0 || row_bytes == 0 || rows > UINT64_MAX / row_bytes) return "invalid";
  Plan p;
  if (!choose_plan(base, rows, row_bytes, out, P_AUTO, &p)) return "invalid";
  return plan_name(p);
}

int ut_set_plan(ut_table* t, const char* name) {
  if (!t || !name) return set_err(UT_EINVAL, "NULL argument");
  if (!strcmp(name, "timing=on") || !strcmp(name, "timing=off")) {
    t->timing = name[8] == 'n';
    return UT_OK;
  }
  if (!strncmp(name, "runs=", 5)) {
    const char* v = name + 5;
    if (!strcmp(v, "auto")) t->runs = -1;
    else if (!strcmp(v, "on")) t->runs = 1;
    else if (!strcmp(v, "off")) t->runs = 0;
    else return set_err(UT_EINVAL, "runs must be auto|on|off, got '%s'", v);
    return UT_OK;
  }
  if (!strncmp(name, "share=", 6)) {
    const char* v = name + 6;
    if (!strcmp(v, "auto")) t->share = -1;
    else if (!strcmp(v, "on")) t->share = 1;
    else if (!strcmp(v, "off")) t->share = 0;
    else return set_err(UT_EINVAL, "share must be auto|on|off, got '%s'", v);
    return UT_OK;
  }
  if (!strncmp(name, "exact=", 6)) {
    const char* v = name + 6;
    if (!strcmp(v, "auto")) t->exact = -1;
    else if (!strcmp(v, "on")) t->exact = 1;
    else if (!strcmp(v, "off")) t->exact = 0;
    else return set_err(UT_EINVAL, "exact must be auto|on|off, got '%s'", v);
    return UT_OK;
  }
  if (!strncmp(name, "stage=", 6)) {
    const char* v = name + 6;
    if (!strcmp(v, "auto")) t->stage = -1;
    else if (!strcmp(v, "on")) t->stage = 1;
    else if (!strcmp(v, "off")) t->stage = 0;
    else return set_err(UT_EINVAL, "stage must be auto|on|off, got '%s'", v);
    return UT_OK;
  }
  if (!strncmp(name, "conc=", 5)) {
    const char* v = name + 5;
    if (!strcmp(v, "auto")) t->conc = -1;
    else if (!strcmp(v, "dense")) t->conc = 0;
    else if (!strcmp(v, "sparse")) t->conc = 1;
    else return set_err(UT_EINVAL, "conc must be auto|dense|sparse, got '%s'", v);
    return UT_OK;
  }
  if (!strncmp(name, "reorder=", 8)) {
    const char* v = name + 8;
    if (!strcmp(v, "auto")) t->reorder = -1;
    else if (!strcmp(v, "on")) t->reorder = 1;
    else if (!strcmp(v, "off")) t->reorder = 0;
    else return set_err(UT_EINVAL, "reorder must be auto|on|off, got '%s'", v);
    return UT_OK;
  }
  bool ok;
  PlanKind k = parse_plan(name, &ok);
  if (!ok) return set_err(UT_EINVAL, "unknown plan '%s'", name);
  Plan p;
  if (k != P_AUTO && !choose_plan((uint64_t)t->host, t->rows, t->rb, 0, k, &p))
    return set_err(UT_EINVAL, "plan '%s' not admissible for this table", name);
  t->forced = k;
  return UT_OK;
}

int ut_get_stats(const ut_table* t, ut_stats* st, int reset) {
  if (!t || !st) return set_err(UT_EINVAL, "NULL argument");
  DevState* s;
  int rc = dev_state(t, &s);
  if (rc != UT_OK) return rc;
  std::lock_guard<std::mutex> lk(s->tmu);
  for (auto& ev : s->pending) {
    cudaError_t e = cudaEventSynchronize(ev.second);
    if (e != cudaSuccess) return cuda_err(e, "cudaEventSynchronize");
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev.first, ev.second);
    s->timed_ms += ms;
    s->timed += 1;
    s->spare.push_back(ev);
  }
  s->pending.clear();
  st->gathers = s->gathers;
  st->kernel_launches = s->launches;
  st->rows = s->rows;
  st->bytes = s->bytes;
  st->timed_launches = s->timed;
  st->gather_kernel_ms = s->timed_ms;
  st->share_gathers = s->shared;
  if (reset) {
    s->shared = 0;
    s->gathers = 0;
    s->launches = 0;
    s->rows = 0;
    s->bytes = 0;
    s->timed = 0;
    s->timed_ms = 0.0;
  }
  return UT_OK;
}

int ut_mem_advise(const ut_table* t, int advice, int device) {
  if (!t) return set_err(UT_EINVAL, "table is NULL");
  static const cudaMemoryAdvise kinds[] = {
      cudaMemAdviseSetPreferredLocation, cudaMemAdviseUnsetPreferredLocation,
      cudaMemAdviseSetAccessedBy,        cudaMemAdviseUnsetAccessedBy,
      cudaMemAdviseSetReadMostly,        cudaMemAdviseUnsetReadMostly};
  if (advice < 0 || advice > 5) return set_err(UT_EINVAL, "unknown advice %d", advice);
  cudaMemLocation loc{};
  if (device < 0) {
    loc.type = cudaMemLocationTypeHost;
    loc.id = 0;
  } else {
    loc.type = cudaMemLocationTypeDevice;
    loc.id = device;
  }
  cudaError_t e = cudaMemAdvise(t->host, t->bytes, kinds[advice], loc);
  cudaGetLastError();
  return (int)e;
}

}  // extern "C"

namespace {
// SetPreferredLocation = host NUMA node node_of(k) for stripe k of `chunk` bytes (k = 0, 1, ...),
// then read the placement back on the first stripe of each of the first `check` stripes; on any
// refusal or silent non-application the whole table is advised back to CPU (ut_create's state).
template <typename NodeOf>
int numa_advise(const ut_table* t, uint64_t chunk, uint64_t check, NodeOf node_of) {
  auto restore = [&] {
    cudaMemLocation cpu{};
    cpu.type = cudaMemLocationTypeHost;
    cpu.id = 0;
    cudaMemAdvise(t->host, t->bytes, cudaMemAdviseSetPreferredLocation, cpu);
    cudaGetLastError();
  };
  uint64_t k = 0;
  for (uint64_t off = 0; off < t->bytes; off += chunk, ++k) {
    cudaMemLocation loc{};
    loc.type = cudaMemLocationTypeHostNuma;
    loc.id = node_of(k);
    const cudaError_t e = cudaMemAdvise(t->host + off, std::min(chunk, t->bytes - off),
                                        cudaMemAdviseSetPreferredLocation, loc);
    if (e != cudaSuccess) {
      cudaGetLastError();
      restore();
      return cuda_err(e, "cudaMemAdvise(SetPreferredLocation = host NUMA node)");
    }
  }
  // Read the advice back: a driver can accept a host-NUMA location and not apply it (measured on
  // this pool's virtualised GPU boxes: cudaSuccess, then no preferred location at all), and a
  // table whose placement silently stayed elsewhere must not be reported as placed.
  for (uint64_t j = 0; j < std::min<uint64_t>(k, check); ++j) {
    const uint64_t off = j * chunk;
    int typ = -1, id = -1;
    const uint64_t len = std::min<uint64_t>(4096, t->bytes - off);
    if (cudaMemRangeGetAttribute(&typ, 4, cudaMemRangeAttributePreferredLocationType,
                                 t->host + off, len) != cudaSuccess ||
        cudaMemRangeGetAttribute(&id, 4, cudaMemRangeAttributePreferredLocationId, t->host + off,
                                 len) != cudaSuccess ||
        typ != (int)cudaMemLocationTypeHostNuma || id != node_of(j)) {
      cudaGetLastError();
      restore();
      return set_err(UT_ENOTSUP, "the driver accepted SetPreferredLocation = host NUMA node %d but "
                     "reports location type %d id %d for stripe %llu: host-NUMA placement is not "
                     "available here (the table keeps SetPreferredLocation = CPU)",
                     node_of(j), typ, id, (unsigned long long)j);
    }
  }
  return UT_OK;
}
}  // namespace

extern "C" {

int ut_numa_interleave(const ut_table* t, int nodes, uint64_t chunk_bytes) {
  if (!t) return set_err(UT_EINVAL, "table is NULL");
  if (nodes < 1) return set_err(UT_EINVAL, "nodes must be >= 1 (got %d)", nodes);
  if (t->alloc_kind != UT_ALLOC_MANAGED)
    return set_err(UT_ENOTSUP, "NUMA striping needs a managed table (ut_create UT_ALLOC_MANAGED)");
  constexpr uint64_t kBlock = 2ull << 20;
  const uint64_t chunk = chunk_bytes == 0 ? kBlock : (chunk_bytes + kBlock - 1) / kBlock * kBlock;
  return numa_advise(t, chunk, (uint64_t)nodes, [nodes](uint64_t k) { return (int)(k % (uint64_t)nodes); });
}

int ut_numa_place(const ut_table* t, int node) {
  if (!t) return set_err(UT_EINVAL, "table is NULL");
  if (node < 0) return set_err(UT_EINVAL, "node must be >= 0 (got %d)", node);
  if (t->alloc_kind != UT_ALLOC_MANAGED)
    return set_err(UT_ENOTSUP, "NUMA placement needs a managed table (ut_create UT_ALLOC_MANAGED)");
  // one advice over the whole range; its placement read back at the first page
  return numa_advise(t, t->bytes, 1, [node](uint64_t) { return node; });
}

int ut_table_get_info(const ut_table* t, ut_table_info* info) {
  if (!t || !info) return set_err(UT_EINVAL, "NULL argument");
  info->rows = t->rows;
  info->row_bytes = t->rb;
  info->host_addr = (uint64_t)t->host;
  const DevState& s = t->dev[t->device];
  info->dev_addr = s.init ? s.dev_base : 0;
  info->registered = t->registered;
  info->alloc_kind = t->alloc_kind;
  info->read_only = t->read_only;
  info->base_mod128 = (int)((uint64_t)t->host & 127);
  info->device = t->device;
  return UT_OK;
}

}  // extern "C"
