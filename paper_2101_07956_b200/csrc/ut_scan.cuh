// ut_scan.cuh — device-wide exclusive scan of uint32 with the length in device memory (used by
// the sampler and by the run-merge reorder). Internal linkage: each translation unit gets its own
// copy of the kernels.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

namespace {

// ---- exclusive scan of uint32 (3 phases: block scans, scan of block sums, add) ---------------
constexpr int kScanBlock = 1024;
constexpr int kScanItems = 4;                       // per thread
constexpr int kScanTile = kScanBlock * kScanItems;  // elements per block

__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* total) {
  __shared__ uint32_t warp_sums[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[w] = x;
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    uint32_t s = lane < nw ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) warp_sums[lane] = s;
  }
  __syncthreads();
  const uint32_t before = w ? warp_sums[w - 1] : 0u;
  *total = warp_sums[(blockDim.x >> 5) - 1];
  __syncthreads();
  return before + x - v;
}

// exclusive scan of in[0 .. *m) -> out, grand total -> *total; launched for m_cap elements
__global__ void __launch_bounds__(kScanBlock) k_scan_tiles(const uint32_t* __restrict__ in, const uint64_t* m_dev,
                                                         uint32_t* __restrict__ out,
                                                         uint32_t* __restrict__ tile_sums) {
  const uint64_t m = *m_dev;
  const uint64_t t0 = (uint64_t)blockIdx.x * kScanTile + (uint64_t)threadIdx.x * kScanItems;
  uint32_t v[kScanItems], sum = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = t0 + k < m ? in[t0 + k] : 0u;
    sum += v[k];
  }
  uint32_t total;
  uint32_t run = block_exclusive_scan(sum, &total);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    if (t0 + k < m) out[t0 + k] = run;
    run += v[k];
  }
  if (threadIdx.x == 0) tile_sums[blockIdx.x] = total;
}

// One block: exclusive scan of the tile sums in place, grand total to *total.
__global__ void __launch_bounds__(kScanBlock) k_scan_sums(uint32_t* sums, const uint64_t* m_dev,
                                                        uint64_t* total) {
  const uint64_t ntiles = (*m_dev + kScanTile - 1) / kScanTile;
  uint32_t carry = 0;
  for (uint64_t b0 = 0; b0 < ntiles; b0 += kScanBlock) {
    const uint64_t i = b0 + threadIdx.x;
    const uint32_t v = i < ntiles ? sums[i] : 0u;
    uint32_t chunk;
    const uint32_t ex = block_exclusive_scan(v, &chunk);
    if (i < ntiles) sums[i] = carry + ex;
    carry += chunk;
  }
  if (threadIdx.x == 0) *total = carry;
}

__global__ void k_scan_add(uint32_t* out, const uint64_t* m_dev, const uint32_t* __restrict__ sums) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < *m_dev && i >= (uint64_t)kScanTile) out[i] += sums[i / kScanTile];
}

inline int scan_blocks_for(uint64_t n, int per = 256) { return (int)std::max<uint64_t>(1, (n + per - 1) / per); }

// exclusive scan of in[0 .. *m_dev) into out (launch sized for m_cap), total into *total_dev
void scan_u32(const uint32_t* in, uint32_t* out, const uint64_t* m_dev, uint64_t m_cap,
              uint64_t* total_dev, uint32_t* tile_sums, cudaStream_t st) {
  const uint64_t ntiles = std::max<uint64_t>(1, (m_cap + kScanTile - 1) / kScanTile);
  k_scan_tiles<<<(int)ntiles, kScanBlock, 0, st>>>(in, m_dev, out, tile_sums);
  k_scan_sums<<<1, kScanBlock, 0, st>>>(tile_sums, m_dev, total_dev);
  if (m_cap > kScanTile) k_scan_add<<<scan_blocks_for(m_cap), 256, 0, st>>>(out, m_dev, tile_sums);
}

}  // namespace
