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

}  // namespace utx
