// ut_internal.h — helpers shared by the library's translation units (not part of the C ABI).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <utility>
#include <vector>

namespace utx {

// Thread-local last error (ut_last_error); both return `code`.
int set_err(int code, const char* fmt, ...);
int cuda_err(cudaError_t e, const char* what);

// Host memory made GPU-addressable in place: adopted when already page-locked and mapped,
// otherwise cudaHostRegister(Portable|Mapped[|ReadOnly]) of the page-aligned range.
struct Pin {
  const uint8_t* base = nullptr;   // page-aligned range covering the caller's bytes
  uint64_t len = 0;
  std::vector<std::pair<const uint8_t*, uint64_t>> regs;   // what we registered (unpin_host
                                                           // unregisters); the rest is adopted
  int read_only = 0;               // 1: every page registered here with cudaHostRegisterReadOnly
  int registered() const { return regs.empty() ? 0 : 1; }
};
int pin_host(const void* p, uint64_t bytes, bool read_only, Pin* out);
void unpin_host(Pin* pin);
// Device address of host address `p` inside `pin` on the current device.
int pin_device_ptr(const Pin& pin, const void* p, uint64_t* dev);

// Host allocations of a ut_alloc_kind (PINNED, MANAGED with the paper's advice, SYSTEM) on
// device `dev`: what ut_create and the recycling pool (ut_pool.cu) both call.
int backend_alloc(int kind, int dev, uint64_t bytes, void** out);
void backend_free(int kind, void* p);

}  // namespace utx

struct ut_pool;

namespace utx {

// The recycling pool's block interface (ut_pool.cu): take returns a block of >= bytes (capacity
// in *cap), give caches it again; pool tables (ut_pool_table) hold one block each.
int pool_take(ut_pool* p, uint64_t bytes, void** out, uint64_t* cap);
int pool_give(ut_pool* p, void* block);
int pool_kind(const ut_pool* p);
int pool_device(const ut_pool* p);

}  // namespace utx
