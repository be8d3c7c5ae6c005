// ut_kernels.cuh — sm_100a gather kernels of the unified-tensor gather (include/ut.h).
//
// Every kernel computes out[i*rb .. (i+1)*rb) = table[idx[i]*rb .. (idx[i]+1)*rb) for i < n,
// reading the table through its device mapping of host memory (Fig. 2b) and
// writing HBM. They differ only in how threads are mapped to bytes:
//
//   narrow<T>      rb in {1,2,4,8}, naturally aligned base and out: one thread per row, one
//                  native-width load and store.
//   vec16<G>       base, rb, out all 16-B aligned and rb <= 512: G lanes per row (G = pow2 >=
//                  rb/16), one 16-B load + store per lane, U rows per group in flight.
//   vec16x         as vec16 with rb > 512: one warp per row, the warp's 16-B windows aligned to
//                  128-B lines (each LDG.128 instruction covers exactly 4 whole lines, the B200
//                  form of the paper's "aligned and merged to the GPU cacheline (128-byte)
//                  granularity"), U instructions in flight per lane.
//   realign<G>     any alignment, rows spanning <= G 16-B chunks: lanes load the row's
//                  16-B-aligned source chunks, exchange neighbours with __shfl_sync and funnel-
//                  shift them onto the destination's 16-B grid (the paper's "output indices are
//                  also identically adjusted"), 16-B stores inside the row and
//                  narrow stores for the two partial edge chunks.
//   realignx       any alignment, wide rows: warp per row, 128-B aligned source windows, a
//                  one-chunk carry between iterations.
//
// Reads never touch table bytes outside [tbase, tend): a 16-B chunk that straddles the table's
// first or last byte is read byte by byte (CLIP variants; only possible when the table's base or
// end is not 16-B aligned). An index < 0 or >= rows zero-fills its row and atomicMin's its
// position into *err (reading R4).
#pragma once
#include <cuda.h>

#include <cstdint>

#ifndef UT_MINB
#define UT_MINB 1
#endif

namespace ut {

struct V4 {
  uint32_t x, y, z, w;
};

__device__ __forceinline__ V4 v4_zero() { return V4{0u, 0u, 0u, 0u}; }

#ifndef UT_LDHINT
#define UT_LDHINT 0
#endif
#if UT_LDHINT == 1
#define UT_LD16 "ld.global.nc.L1::no_allocate.L2::128B.v4.u32"
#elif UT_LDHINT == 2
#define UT_LD16 "ld.global.nc.L1::no_allocate.L2::256B.v4.u32"
#elif UT_LDHINT == 3
#define UT_LD16 "ld.global.v4.u32"
#elif UT_LDHINT == 4
#define UT_LD16 "ld.global.nc.L1::no_allocate.L2::64B.v4.u32"
#else
#define UT_LD16 "ld.global.nc.L1::no_allocate.v4.u32"
#endif

// 16-B load from the device-mapped host table. Non-coherent path, no L1 allocation: the table
// is read-only for the duration of a gather and every byte is used once per request.
__device__ __forceinline__ V4 ld_table16(uint64_t a) {
  V4 v;
  asm(UT_LD16 " {%0, %1, %2, %3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(a));
  return v;
}

__device__ __forceinline__ uint32_t ld_table_u8(uint64_t a) {
  uint16_t v;
  asm("ld.global.nc.u8 %0, [%1];" : "=h"(v) : "l"(a));
  return v;
}

// 16-B chunk at a (16-B aligned) of which only the bytes in [lo, hi) may be read; the rest are 0.
__device__ __noinline__ V4 ld_table16_clipped(uint64_t a, uint64_t lo, uint64_t hi) {
  uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
  for (int b = 0; b < 16; ++b) {
    uint64_t p = a + b;
    if (p >= lo && p < hi) w[b >> 2] |= ld_table_u8(p) << ((b & 3) * 8);
  }
  return V4{w[0], w[1], w[2], w[3]};
}

template <bool CLIP>
__device__ __forceinline__ V4 ld_chunk(uint64_t a, uint64_t tbase, uint64_t tend) {
  if (CLIP && (a < tbase || a + 16 > tend)) return ld_table16_clipped(a, tbase, tend);
  return ld_table16(a);
}

__device__ __forceinline__ void st16(uint64_t a, V4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(a), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Store bytes [lo, hi) of the 16-B value v to the 16-B aligned address D (+lo), using the widest
// naturally aligned pieces. Only the two edge chunks of a row take this path.
__device__ __noinline__ void st_partial(uint64_t D, V4 v, int lo, int hi) {
  uint64_t w0 = (uint64_t)v.x | ((uint64_t)v.y << 32);
  uint64_t w1 = (uint64_t)v.z | ((uint64_t)v.w << 32);
  int b = lo;
  while (b < hi) {
    uint64_t w = b < 8 ? w0 : w1;
    int sh = (b & 7) * 8;
    if ((b & 7) == 0 && hi - b >= 8) {
      *reinterpret_cast<uint64_t*>(D + b) = w;
      b += 8;
    } else if ((b & 3) == 0 && hi - b >= 4) {
      *reinterpret_cast<uint32_t*>(D + b) = (uint32_t)(w >> sh);
      b += 4;
    } else if ((b & 1) == 0 && hi - b >= 2) {
      *reinterpret_cast<uint16_t*>(D + b) = (uint16_t)(w >> sh);
      b += 2;
    } else {
      *reinterpret_cast<uint8_t*>(D + b) = (uint8_t)(w >> sh);
      b += 1;
    }
  }
}

// Store the part of the 16-B destination chunk at D (16-B aligned) that lies in [d, dend).
__device__ __forceinline__ void st_chunk_clip(uint64_t D, V4 v, uint64_t d, uint64_t dend) {
  if (D >= d && D + 16 <= dend) {
    st16(D, v);
  } else if (D + 16 > d && D < dend) {
    int lo = D < d ? (int)(d - D) : 0;
    int hi = D + 16 > dend ? (int)(dend - D) : 16;
    st_partial(D, v, lo, hi);
  }
}

// Bytes [r, r+16) of the 32-byte little-endian concatenation lo || hi, r in [0, 16).
__device__ __forceinline__ V4 funnel16(V4 lo, V4 hi, int r) {
  const int q = r >> 2;
  const uint32_t sh = (uint32_t)(r & 3) * 8u;
  uint32_t t0 = q == 0 ? lo.x : q == 1 ? lo.y : q == 2 ? lo.z : lo.w;
  uint32_t t1 = q == 0 ? lo.y : q == 1 ? lo.z : q == 2 ? lo.w : hi.x;
  uint32_t t2 = q == 0 ? lo.z : q == 1 ? lo.w : q == 2 ? hi.x : hi.y;
  uint32_t t3 = q == 0 ? lo.w : q == 1 ? hi.x : q == 2 ? hi.y : hi.z;
  uint32_t t4 = q == 0 ? hi.x : q == 1 ? hi.y : q == 2 ? hi.z : hi.w;
  return V4{__funnelshift_r(t0, t1, sh), __funnelshift_r(t1, t2, sh), __funnelshift_r(t2, t3, sh),
            __funnelshift_r(t3, t4, sh)};
}

__device__ __forceinline__ V4 shfl4(V4 v, int src, int width) {
  return V4{__shfl_sync(0xffffffffu, v.x, src, width), __shfl_sync(0xffffffffu, v.y, src, width),
            __shfl_sync(0xffffffffu, v.z, src, width), __shfl_sync(0xffffffffu, v.w, src, width)};
}

__device__ __forceinline__ V4 shfl4_up1(V4 v) {
  return V4{__shfl_up_sync(0xffffffffu, v.x, 1), __shfl_up_sync(0xffffffffu, v.y, 1),
            __shfl_up_sync(0xffffffffu, v.z, 1), __shfl_up_sync(0xffffffffu, v.w, 1)};
}

struct GatherArgs {
  uint64_t tbase;   // device address of table byte 0
  uint64_t rows;
  uint64_t rb;
  const int64_t* idx;
  uint64_t n;
  uint64_t out;     // device address of out byte 0
  unsigned long long* err;
  const uint32_t* perm;   // optional visiting order (work item j handles output row perm[j])
  const uint64_t* n_dev;  // optional: the row count lives in device memory (min(*n_dev, n))
  const CUtensorMap* tmap = nullptr;   // host copy of the table's tensor map ("tma4" plan only)
  uint64_t pos0 = 0;      // position of idx[0] in the caller's list (chunked gathers' error record)
};

// The kernels' view of the arguments: n read from device memory when the launch is
// size-oblivious (ut_gather_dn: a sampler on the device produced the index list).
__device__ __forceinline__ GatherArgs with_dev_n(const GatherArgs& a) {
  GatherArgs b = a;
  if (a.n_dev) {
    const uint64_t n = *a.n_dev;
    b.n = n < a.n ? n : a.n;
  }
  return b;
}

// Output row handled by work item j: j itself, or perm[j] when the rows are visited in the
// translation-locality order built by k_bucket_* (DESIGN.md §Reorder).
template <bool PERM>
__device__ __forceinline__ uint64_t row_of(const GatherArgs& a, uint64_t j, bool inb) {
  if (!PERM) return j;
  return inb ? (uint64_t)__ldg(a.perm + j) : 0ull;
}

// Position i of this launch's list is out of range: keep the smallest position of the caller's
// whole list (a.pos0 = where this launch's list starts in it, for chunked gathers).
__device__ __forceinline__ void record_bad(const GatherArgs& a, uint64_t i) {
  atomicMin(a.err, (unsigned long long)(a.pos0 + i));
}

// ---------------------------------------------------------------------------------------------
// narrow<T>: one thread per row, U rows per thread in flight.
template <typename T, int U, bool PERM>
__global__ void __launch_bounds__(256, UT_MINB) k_narrow(GatherArgs a_) {
  const GatherArgs a = with_dev_n(a_);
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t t0 = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (uint64_t base = 0; base < a.n; base += nthreads * U) {
    T v[U];
    bool inb[U], ok[U];
    uint64_t ii[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = base + (uint64_t)u * nthreads + t0;
      inb[u] = j < a.n;
      const uint64_t i = ii[u] = row_of<PERM>(a, j, inb[u]);
      int64_t r = inb[u] ? __ldg(a.idx + i) : 0;
      ok[u] = inb[u] && (uint64_t)r < a.rows;
      v[u] = ok[u] ? *reinterpret_cast<const T*>(a.tbase + (uint64_t)r * sizeof(T)) : T(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = ii[u];
      if (inb[u]) {
        *reinterpret_cast<T*>(a.out + i * sizeof(T)) = v[u];
        if (!ok[u]) record_bad(a, i);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Single-pass kernels: G lanes per row, 32/G rows per warp step, U steps in flight per warp tile.
// ALIGNED: base, rb, out 16-B aligned (vec16<G>); else realign<G>.
template <int G, int U, bool ALIGNED, bool CLIP, bool PERM>
__global__ void __launch_bounds__(256, UT_MINB) k_single(GatherArgs a_) {
  const GatherArgs a = with_dev_n(a_);
  constexpr int RPS = 32 / G;          // rows per warp step
  constexpr int RPT = RPS * U;         // rows per warp tile
  const int lane = threadIdx.x & 31;
  const int grp = lane / G;
  const int q = lane % G;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t ntiles = (a.n + RPT - 1) / RPT;
  const uint64_t tend = a.tbase + a.rows * a.rb;

  for (uint64_t tile = warp; tile < ntiles; tile += nwarps) {
    V4 cur[U];
    uint64_t s[U], ii[U];
    bool inb[U], ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = tile * RPT + (uint64_t)u * RPS + grp;
      inb[u] = j < a.n;
      const uint64_t i = ii[u] = row_of<PERM>(a, j, inb[u]);
      const int64_t r = inb[u] ? __ldg(a.idx + i) : 0;
      ok[u] = inb[u] && (uint64_t)r < a.rows;
      s[u] = a.tbase + (ok[u] ? (uint64_t)r : 0ull) * a.rb;
      cur[u] = v4_zero();
      if (ALIGNED) {
        if (ok[u] && (uint64_t)q * 16 < a.rb) cur[u] = ld_table16(s[u] + 16ull * q);
      } else {
        const uint64_t s0 = s[u] & ~15ull;
        const uint64_t A = s0 + 16ull * q;
        if (ok[u] && A < s[u] + a.rb) cur[u] = ld_chunk<CLIP>(A, a.tbase, tend);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = ii[u];
      const uint64_t d = a.out + i * a.rb;
      if (ALIGNED) {
        if (inb[u] && (uint64_t)q * 16 < a.rb) st16(d + 16ull * q, cur[u]);
      } else {
        // destination chunk q of the row sits at D = floor16(d) + 16q; its source bytes start
        // at D + (s - d), i.e. chunk q+koff of the source window at byte offset r.
        const int delta = (int)(s[u] & 15) - (int)(d & 15);
        const int koff = delta < 0 ? -1 : 0;
        const int r = delta & 15;
        const int k = q + koff;
        V4 lo = shfl4(cur[u], k & (G - 1), G);
        V4 hi = shfl4(cur[u], (k + 1) & (G - 1), G);
        if (k < 0) lo = v4_zero();
        if (k + 1 >= G) hi = v4_zero();
        if (inb[u]) {
          const uint64_t D = (d & ~15ull) + 16ull * q;
          st_chunk_clip(D, funnel16(lo, hi, r), d, d + a.rb);
        }
      }
      if (inb[u] && !ok[u] && q == 0) record_bad(a, i);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Multi-pass kernels: one warp per row, the row's source window starts on a 128-B line and is
// walked 32*U chunks at a time (U LDG.128 per lane in flight).
template <int U, bool ALIGNED, bool CLIP, bool PERM>
__global__ void __launch_bounds__(256, UT_MINB) k_multi(GatherArgs a_) {
  const GatherArgs a = with_dev_n(a_);
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t tend = a.tbase + a.rows * a.rb;

  for (uint64_t j = warp; j < a.n; j += nwarps) {
    const uint64_t i = row_of<PERM>(a, j, true);
    const int64_t ridx = __ldg(a.idx + i);
    const bool ok = (uint64_t)ridx < a.rows;
    const uint64_t s = a.tbase + (ok ? (uint64_t)ridx : 0ull) * a.rb;
    const uint64_t send = s + a.rb;
    const uint64_t d = a.out + i * a.rb;
    const uint64_t ws = s & ~127ull;
    const uint64_t we = (send + 15) & ~15ull;
    const uint64_t nch = (we - ws) >> 4;
    if (ALIGNED) {
      for (uint64_t c0 = 0; c0 < nch; c0 += 32 * U) {
        V4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t A = ws + 16ull * (c0 + 32u * u + lane);
          cur[u] = (ok && A >= s && A < send) ? ld_table16(A) : v4_zero();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t A = ws + 16ull * (c0 + 32u * u + lane);
          if (A >= s && A < send) st16(A - s + d, cur[u]);
        }
      }
    } else {
      const int r = (int)((s - d) & 15);
      const uint64_t dend = d + a.rb;
      V4 carry = v4_zero();
      // slot c combines source chunks c-1 and c into the destination chunk
      // D(c) = ws + 16(c-1) + r + (d - s); slots 0..nch cover every destination chunk.
      for (uint64_t c0 = 0; c0 <= nch; c0 += 32 * U) {
        V4 cur[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t c = c0 + 32u * u + lane;
          const uint64_t A = ws + 16ull * c;
          cur[u] = (ok && c < nch && A + 16 > s) ? ld_chunk<CLIP>(A, a.tbase, tend) : v4_zero();
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint64_t c = c0 + 32u * u + lane;
          V4 prev = shfl4_up1(cur[u]);
          if (lane == 0) prev = carry;
          carry = shfl4(cur[u], 31, 32);
          const uint64_t D = ws + 16ull * c - 16ull + (uint64_t)r + d - s;
          st_chunk_clip(D, funnel16(prev, cur[u], r), d, dend);
        }
      }
    }
    if (!ok && lane == 0) record_bad(a, i);
  }
}

// ---------------------------------------------------------------------------------------------
// staged<T>: output rows in mapped HOST memory (ut_gather_host's direct path). A block owns a
// tile of consecutive output rows: it reads the tile's rows from the table into shared memory
// (flattened over the tile's W-byte chunks, U chunks per thread in flight), then writes the tile's
// contiguous output span with coalesced W-byte stores, so the write side of the link sees whole
// 128-B lines except at tile edges instead of two partial lines per row. The hypothesis (rows of
// 400 B reach 29.7 GB/s host->host vs 36.6-39.9 for rows that are whole lines) did not hold: the
// gap is on the read side, and staging gains nothing (opt-in only, "stage=on").
// Requires base, rb and out to be W-aligned (W = sizeof(T)); the tile is <= kStageBytes.
constexpr int kStageBytes = 16384;
constexpr int kStageMaxRows = 1024;

template <typename T>
__device__ __forceinline__ T ld_table_w(uint64_t a);
template <>
__device__ __forceinline__ uint4 ld_table_w<uint4>(uint64_t a) {
  const V4 v = ld_table16(a);
  return make_uint4(v.x, v.y, v.z, v.w);
}
template <>
__device__ __forceinline__ uint2 ld_table_w<uint2>(uint64_t a) {
  uint2 v;
  asm("ld.global.nc.L1::no_allocate.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "l"(a));
  return v;
}
template <>
__device__ __forceinline__ uint32_t ld_table_w<uint32_t>(uint64_t a) {
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(a));
  return v;
}

// The tile sits in shared memory at the output span's offset within its first 128-B line, so
// shared 16-B chunk g is the output's 16-B chunk g counted from that line: every warp store
// instruction then covers 4 whole aligned lines, and only the tile's two edge lines are partial.
template <typename T, int U>
__global__ void __launch_bounds__(256) k_staged(GatherArgs a_, uint32_t tile_rows) {
  const GatherArgs a = with_dev_n(a_);
  __shared__ __align__(128) uint8_t tile[kStageBytes + 128];
  __shared__ uint64_t src[kStageMaxRows];          // per tile row: source address, or ~0 if bad
  constexpr uint32_t W = sizeof(T);
  const uint32_t cpr = (uint32_t)(a.rb / W);       // chunks per row
  const uint64_t ntiles = (a.n + tile_rows - 1) / tile_rows;
  for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint64_t r0 = t * tile_rows;
    const uint32_t nr = (uint32_t)((a.n - r0) < tile_rows ? (a.n - r0) : tile_rows);
    const uint64_t D0 = a.out + r0 * a.rb;
    const uint32_t h = (uint32_t)(D0 & 127);       // a multiple of W
    const uint32_t bytes = nr * (uint32_t)a.rb;
    for (uint32_t k = threadIdx.x; k < nr; k += blockDim.x) {
      const int64_t r = __ldg(a.idx + r0 + k);
      const bool ok = (uint64_t)r < a.rows;
      src[k] = ok ? a.tbase + (uint64_t)r * a.rb : ~0ull;
      if (!ok) record_bad(a, r0 + k);
    }
    __syncthreads();
    const uint32_t nch = nr * cpr;
    T* tl = reinterpret_cast<T*>(tile + h);        // chunk f of the tile = row f / cpr, chunk f % cpr
    for (uint32_t f0 = 0; f0 < nch; f0 += blockDim.x * U) {
      T v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * blockDim.x + threadIdx.x;
        v[u] = T{};
        if (f < nch) {
          const uint32_t row = f / cpr, c = f - row * cpr;
          const uint64_t sa = src[row];
          if (sa != ~0ull) v[u] = ld_table_w<T>(sa + (uint64_t)c * W);
        }
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t f = f0 + u * blockDim.x + threadIdx.x;
        if (f < nch) tl[f] = v[u];
      }
    }
    __syncthreads();
    const uint64_t L0 = D0 - h;                    // the span's first 128-B line
    const uint32_t G = (h + bytes + 15) / 16;
    for (uint32_t g = threadIdx.x; g < G; g += blockDim.x) {
      const uint4 w = reinterpret_cast<const uint4*>(tile)[g];
      const V4 v{w.x, w.y, w.z, w.w};
      const uint32_t lo = 16 * g < h ? h - 16 * g : 0;
      const uint32_t hi = h + bytes - 16 * g < 16 ? h + bytes - 16 * g : 16;
      if (lo == 0 && hi == 16) st16(L0 + 16ull * g, v);
      else st_partial(L0 + 16ull * g, v, (int)lo, (int)hi);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------------------------
// bulk<U>: the row is fetched by the TMA unit (1-D cp.async.bulk global -> shared, completion on an
// mbarrier) instead of by LDG, then stored to HBM from shared memory. Table base, rb and out
// 16-B aligned, rb <= kBulkMaxRow. One warp per row-slot, U rows in flight per warp.
constexpr int kBulkMaxRow = 4096;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t phase) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(phase)
      : "memory");
  return ok != 0;
}

template <int U, bool PERM>
__global__ void __launch_bounds__(256, 1) k_bulk(GatherArgs a_) {
  const GatherArgs a = with_dev_n(a_);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[8 * U];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t rbp = (uint32_t)((a.rb + 127) & ~127ull);
  uint8_t* my = smem + (size_t)wib * U * rbp;
  const uint32_t bar0 = smem_u32(&bars[wib * U]);
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t ntiles = (a.n + U - 1) / U;
  uint32_t phase = 0;
  for (uint64_t tile = warp; tile < ntiles; tile += nwarps) {
    uint32_t issued = 0;
    uint64_t rowi[U];
    bool inb[U];
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = tile * U + u;
      inb[u] = j < a.n;
      const uint64_t i = rowi[u] = row_of<PERM>(a, j, inb[u]);
      const int64_t r = inb[u] ? __ldg(a.idx + i) : 0;
      const bool ok = inb[u] && (uint64_t)r < a.rows;
      if (ok) issued |= 1u << u;
      if (lane == 0 && ok) {
        const uint32_t bar = bar0 + 8u * u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)a.rb)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_u32(my + (size_t)u * rbp)),
            "l"(a.tbase + (uint64_t)r * a.rb), "r"((uint32_t)a.rb), "r"(bar)
            : "memory");
      }
      if (lane == 0 && inb[u] && !ok) record_bad(a, i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!inb[u]) continue;
      const uint64_t d = a.out + rowi[u] * a.rb;
      if (issued & (1u << u)) {
        while (!mbar_try_wait(bar0 + 8u * u, phase)) {
        }
        for (uint32_t c = lane * 16; c < a.rb; c += 32 * 16)
          st16(d + c, *reinterpret_cast<const V4*>(my + (size_t)u * rbp + c));
      } else {
        for (uint32_t c = lane * 16; c < a.rb; c += 32 * 16) st16(d + c, v4_zero());
      }
    }
    // every issued barrier completed one phase; barriers not issued stay in the old phase, so
    // re-align them by arriving once (count 1) to keep one phase bit for all slots.
    if (lane == 0) {
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (!(issued & (1u << u)))
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar0 + 8u * u) : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!(issued & (1u << u))) {
        while (!mbar_try_wait(bar0 + 8u * u, phase)) {
        }
      }
    }
    phase ^= 1u;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------
// tma4<U>: the TMA unit's row gather (cp.async.bulk.tensor.2d ... tile::gather4): one instruction
// fetches 4 rows of the table, viewed as a 2-D tensor of rows x (rb/4) 32-bit words, into shared
// memory; the warp then stores them to HBM. A/B plan only (SURVEY §7 step 4 "TMA tile::gather4 for
// rb % 16 == 0 tables"). rb % 16 == 0, rb <= 1024 (box width <= 256 words), rows < 2^31. Rows
// past n, and bad indices (mapped to the out-of-bounds coordinate `rows`), are zero-filled by the
// TMA unit without touching memory. One warp per group of 4 rows, U groups in flight per warp.
constexpr int kTma4MaxRow = 1024;

template <int U>
__global__ void __launch_bounds__(128, 1) k_tma4(const __grid_constant__ CUtensorMap tm, GatherArgs a_) {
  const GatherArgs a = with_dev_n(a_);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t bars[4 * U];
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const uint32_t slot = (uint32_t)((4 * a.rb + 127) & ~127ull);
  uint8_t* my = smem + (size_t)wib * U * slot;
  const uint32_t bar0 = smem_u32(&bars[wib * U]);
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t ngroups = (a.n + 3) / 4;
  const uint64_t ntiles = (ngroups + U - 1) / U;
  uint32_t phase = 0;
  for (uint64_t tile = warp; tile < ntiles; tile += nwarps) {
    if (lane == 0) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = tile * U + u;
      // lanes 0..3 read the group's 4 indices; lane 0 issues the gather (always, so every
      // barrier completes one phase per tile; rows past n use the out-of-bounds coordinate)
      int32_t crd = (int32_t)a.rows;
      if (lane < 4) {
        const uint64_t i = g * 4 + lane;
        if (i < a.n) {
          const int64_t r = __ldg(a.idx + i);
          if ((uint64_t)r < a.rows) crd = (int32_t)r;
          else record_bad(a, i);
        }
      }
      const int32_t c0 = __shfl_sync(0xffffffffu, crd, 0), c1 = __shfl_sync(0xffffffffu, crd, 1);
      const int32_t c2 = __shfl_sync(0xffffffffu, crd, 2), c3 = __shfl_sync(0xffffffffu, crd, 3);
      if (lane == 0) {
        const uint32_t bar = bar0 + 8u * u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((uint32_t)(4 * a.rb))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(my + (size_t)u * slot)),
            "l"(&tm), "r"(0), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar)
            : "memory");
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t g = tile * U + u;
      while (!mbar_try_wait(bar0 + 8u * u, phase)) {
      }
      const uint64_t i0 = g * 4;
      const uint64_t nr = i0 < a.n ? (a.n - i0 < 4 ? a.n - i0 : 4) : 0;
      const uint32_t bytes = (uint32_t)(nr * a.rb);
      for (uint32_t c = lane * 16; c < bytes; c += 32 * 16)
        st16(a.out + i0 * a.rb + c, *reinterpret_cast<const V4*>(my + (size_t)u * slot + c));
    }
    phase ^= 1u;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------------------------
// The paper's own indexing kernels, for the ablation only (never auto-selected):
//   paper_naive — PyTorch's stock index kernel as PAPER.md:557-558 describes it: one thread per
//                 4-B feature, rows contiguous in thread space (thread r*W + j copies element j
//                 of row idx[r] to output element r*W + j).
//   paper_shift — the circular shift of PAPER.md:562-566 (reading R13): thread j of row r copies
//                 element (j + s_r) mod W with s_r = (r*W - idx[r]*W) mod 32, writing the same
//                 rotated output position ("the output indices are also identically adjusted").
// Both need rb % 4 == 0 and 4-B aligned base and out. W = rb / 4.
template <bool SHIFT>
__global__ void __launch_bounds__(256) k_paper(GatherArgs a_) {
  const GatherArgs a = with_dev_n(a_);
  const uint64_t W = a.rb >> 2;
  const uint64_t total = a.n * W;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const uint64_t r = t / W;
    const uint64_t j = t - r * W;
    const int64_t g = __ldg(a.idx + r);
    const bool ok = (uint64_t)g < a.rows;
    uint64_t e = j;
    if (SHIFT) {
      const uint64_t s = ((r * W) - ((uint64_t)(ok ? g : 0) * W)) & 31ull;   // mod L = 32
      e = j + s;
      if (e >= W) e -= W;      // "adding or subtracting the length of the node feature"
      if (e >= W) e %= W;      // (only when W < 32)
    }
    uint32_t v = 0;
    if (ok) v = __ldg(reinterpret_cast<const uint32_t*>(a.tbase) + (uint64_t)g * W + e);
    reinterpret_cast<uint32_t*>(a.out)[r * W + e] = v;
    if (!ok && j == 0) record_bad(a, r);
  }
}

// ---------------------------------------------------------------------------------------------
// Translation-locality reorder: a counting sort of the work items by the table
// region (1 << shift bytes, at most kMaxBuckets regions) their row starts in. The visiting order
// changes, the result does not: every work item still writes its own output row.
// Each block owns a contiguous chunk of work items and keeps a shared-memory histogram, so global
// atomics are one per (block, non-empty bucket) instead of one per item.
constexpr int kMaxBuckets = 32768;   // 128 KiB of dynamic shared memory per block

__device__ __forceinline__ uint32_t bucket_of(const GatherArgs& a, uint64_t i, int shift) {
  const int64_t r = __ldg(a.idx + i);
  return (uint64_t)r < a.rows ? (uint32_t)(((uint64_t)r * a.rb) >> shift) : 0u;
}

__global__ void __launch_bounds__(512) k_bucket_count(GatherArgs a_, int shift, uint32_t nb,
                                                      uint64_t chunk, uint32_t* cnt) {
  const GatherArgs a = with_dev_n(a_);
  extern __shared__ uint32_t hist[];    // nb entries
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0u;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(a.n, lo + chunk);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&hist[bucket_of(a, i, shift)], 1u);
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x)
    if (hist[b]) atomicAdd(cnt + b, hist[b]);
}

// In-place exclusive scan of cnt[0..nb) by one block of 1024 threads: the counts are staged in
// shared memory with coalesced loads, each thread scans a contiguous run, runs are combined with
// a block-wide scan, and the result is written back coalesced.
__global__ void __launch_bounds__(1024) k_bucket_scan(uint32_t* cnt, uint32_t nb) {
  extern __shared__ uint32_t v[];       // nb entries
  __shared__ uint32_t part[1024];
  for (uint32_t k = threadIdx.x; k < nb; k += 1024) v[k] = cnt[k];
  __syncthreads();
  const uint32_t per = (nb + 1023) / 1024;
  const uint32_t lo = min(nb, threadIdx.x * per), hi = min(nb, lo + per);
  uint32_t sum = 0;
  for (uint32_t k = lo; k < hi; ++k) sum += v[k];
  part[threadIdx.x] = sum;
  __syncthreads();
  for (uint32_t off = 1; off < 1024; off <<= 1) {
    uint32_t x = threadIdx.x >= off ? part[threadIdx.x - off] : 0u;
    __syncthreads();
    part[threadIdx.x] += x;
    __syncthreads();
  }
  uint32_t run = part[threadIdx.x] - sum;
  for (uint32_t k = lo; k < hi; ++k) {
    const uint32_t c = v[k];
    v[k] = run;
    run += c;
  }
  __syncthreads();
  for (uint32_t k = threadIdx.x; k < nb; k += 1024) cnt[k] = v[k];
}

__global__ void __launch_bounds__(512) k_bucket_scatter(GatherArgs a_, int shift, uint32_t nb,
                                                        uint64_t chunk, uint32_t* cursor,
                                                        uint32_t* perm) {
  const GatherArgs a = with_dev_n(a_);
  extern __shared__ uint32_t hist[];    // nb entries
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) hist[b] = 0u;
  __syncthreads();
  const uint64_t lo = (uint64_t)blockIdx.x * chunk;
  const uint64_t hi = min(a.n, lo + chunk);
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) atomicAdd(&hist[bucket_of(a, i, shift)], 1u);
  __syncthreads();
  // reserve this block's range in every non-empty bucket; hist[b] becomes the range start
  for (uint32_t b = threadIdx.x; b < nb; b += blockDim.x) {
    const uint32_t c = hist[b];
    if (c) hist[b] = atomicAdd(cursor + b, c);
  }
  __syncthreads();
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x)
    perm[atomicAdd(&hist[bucket_of(a, i, shift)], 1u)] = (uint32_t)i;
}

// ---------------------------------------------------------------------------------------------
// Run merge: with the work items in exact table order, rows that are neighbours in
// the table form runs; one warp copies a run's contiguous byte span through 128-B-aligned windows,
// so the line two adjacent rows share is requested once instead of twice (two partial requests).
// Only for 16-B aligned tables and outputs with rb % 16 == 0: a 16-B chunk then lies in one row.

// int32 row ids -> int64 (ut_gather_i32): sign extension, so a negative id stays out of range.
__global__ void __launch_bounds__(256) k_widen_i32(const int32_t* __restrict__ in, int64_t* __restrict__ out,
                                                   uint64_t n) {
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = (int64_t)__ldg(in + i);
}

// Exact order inside each (small) bucket: one thread insertion-sorts its bucket's work items by
// row id. ends[] = bucket ends after k_bucket_scatter. Buckets above 256 items are left as they
// are (order only affects how many runs are found, never the result).
__global__ void __launch_bounds__(256) k_bucket_sort(GatherArgs a_, const uint32_t* __restrict__ ends,
                                                     uint32_t nb, uint32_t* perm) {
  const GatherArgs a = with_dev_n(a_);
  const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nb) return;
  const uint32_t lo = b ? ends[b - 1] : 0u, hi = ends[b];
  if (hi - lo < 2 || hi - lo > 256) return;
  for (uint32_t x = lo + 1; x < hi; ++x) {
    const uint32_t item = perm[x];
    const uint64_t key = (uint64_t)__ldg(a.idx + item);
    uint32_t y = x;
    while (y > lo && (uint64_t)__ldg(a.idx + perm[y - 1]) > key) {
      perm[y] = perm[y - 1];
      --y;
    }
    perm[y] = item;
  }
}

// flags[j] = 1 where work item j starts a run (its row is not the successor of item j-1's row).
__global__ void __launch_bounds__(256) k_run_flags(GatherArgs a_, uint32_t* __restrict__ flags) {
  const GatherArgs a = with_dev_n(a_);
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  const uint64_t r = (uint64_t)__ldg(a.idx + a.perm[j]);
  uint32_t start = 1u;
  if (j > 0 && r < a.rows) {
    const uint64_t rp = (uint64_t)__ldg(a.idx + a.perm[j - 1]);
    start = (rp < a.rows && r == rp + 1) ? 0u : 1u;
  }
  flags[j] = start;
}

// *out = the effective row count: min(*n_dev, n) when the count lives on the device, else n.
__global__ void k_eff_n(const uint64_t* n_dev, uint64_t n, uint64_t* out) {
  *out = (n_dev && *n_dev < n) ? *n_dev : n;
}

// run_start[pos[j]] = j for run starts; run_start[n_runs] = n.
__global__ void __launch_bounds__(256) k_run_emit(GatherArgs a_, const uint32_t* __restrict__ flags,
                                                  const uint32_t* __restrict__ pos,
                                                  const uint64_t* n_runs, uint32_t* run_start) {
  const GatherArgs a = with_dev_n(a_);
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= a.n) return;
  if (flags[j]) run_start[pos[j]] = (uint32_t)j;
  if (j == 0) run_start[*n_runs] = (uint32_t)a.n;
}

template <int U>
__global__ void __launch_bounds__(256) k_runs(GatherArgs a_, const uint32_t* __restrict__ run_start,
                                              const uint64_t* n_runs) {
  const GatherArgs a = with_dev_n(a_);
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t nr = *n_runs;
  for (uint64_t run = warp; run < nr; run += nwarps) {
    const uint32_t j0 = run_start[run], j1 = run_start[run + 1];
    const uint64_t i0 = a.perm[j0];
    const uint64_t r0 = (uint64_t)__ldg(a.idx + i0);
    if (r0 >= a.rows) {        // an out-of-range index is a run of one: zero row + record
      const uint64_t d = a.out + i0 * a.rb;
      for (uint64_t c = (uint64_t)lane * 16; c < a.rb; c += 32 * 16) st16(d + c, v4_zero());
      if (lane == 0) record_bad(a, i0);
      continue;
    }
    const uint64_t s = a.tbase + r0 * a.rb;
    const uint64_t send = s + (uint64_t)(j1 - j0) * a.rb;
    const uint64_t ws = s & ~127ull;
    const uint64_t nch = (((send + 15) & ~15ull) - ws) >> 4;
    for (uint64_t c0 = 0; c0 < nch; c0 += 32 * U) {
      V4 cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t A = ws + 16ull * (c0 + 32u * u + lane);
        cur[u] = (A >= s && A < send) ? ld_table16(A) : v4_zero();
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t A = ws + 16ull * (c0 + 32u * u + lane);
        if (A >= s && A < send) {
          const uint64_t rel = A - s;
          const uint64_t k = rel / a.rb;
          st16(a.out + (uint64_t)a.perm[j0 + k] * a.rb + (rel - k * a.rb), cur[u]);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Neighbour line sharing ("share", vec16 tables with 128 < rb <= 512). Selected
// rows r and r+1 whose boundary does not fall on a 128-B line both touch that line; fetched by
// both warps it costs two sysmem requests, and at these widths the request count, not the bytes,
// bounds the link. k_share_mark gives every selected row one canonical work item
// (any one occurrence of a duplicated row wins) in a per-gather hash of the selection, O(n):
// 2^bits >= 2n slots of one 64-bit word, (r + 1) << 32 | (i + 1), open addressing with linear
// probing, 0 = empty. In k_share the warp of row r also loads the bytes of row r+1 that lie in r's
// last line and stores them into row r+1's canonical output row; that canonical item skips its
// first (shared) line. Both sides decide from the same table — fixed for the whole gather — so
// every output byte is written by its own row's warp or by a predecessor's warp that read the
// same table bytes (duplicates of r write identical bytes). The result is the plain gather
// (oracle), unchanged.
struct ShareHash {
  unsigned long long* slots;
  uint32_t bits;
  __device__ __forceinline__ uint64_t home(uint64_t r) const {
    return (r * 0x9E3779B97F4A7C15ull) >> (64 - bits);
  }
  // canonical work item + 1 of row r, 0 when r is not selected
  __device__ __forceinline__ uint32_t find(uint64_t r) const {
    const uint64_t mask = (1ull << bits) - 1, key = r + 1;
    for (uint64_t h = home(r);; h = (h + 1) & mask) {
      const unsigned long long w = __ldcg(slots + h);
      if (w == 0ull) return 0u;
      if ((w >> 32) == key) return (uint32_t)w;
    }
  }
};

__global__ void __launch_bounds__(256) k_share_mark(GatherArgs a_, ShareHash hs) {
  const GatherArgs a = with_dev_n(a_);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t mask = (1ull << hs.bits) - 1;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride) {
    const int64_t r = __ldg(a.idx + i);
    if ((uint64_t)r >= a.rows) continue;
    const unsigned long long w = ((unsigned long long)(r + 1) << 32) | (uint32_t)(i + 1);
    for (uint64_t h = hs.home((uint64_t)r);; h = (h + 1) & mask) {
      const unsigned long long old = atomicCAS(hs.slots + h, 0ull, w);
      if (old == 0ull || (old >> 32) == (unsigned long long)(r + 1)) break;
    }
  }
}

// One warp per row step, U steps in flight per warp; lane q moves 16-B chunk q (and q + 32 when
// TWO, rows > 400 B) of the byte range [lo, hi) relative to the row start: lo skips the shared
// first line, hi extends over the successor's bytes in the last line.
template <int U, bool TWO>
__global__ void __launch_bounds__(256, UT_MINB) k_share(GatherArgs a_, ShareHash hs) {
  const GatherArgs a = with_dev_n(a_);
  constexpr int C = TWO ? 2 : 1;
  const int lane = threadIdx.x & 31;
  const uint64_t warp = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t ntiles = (a.n + U - 1) / U;
  for (uint64_t tile = warp; tile < ntiles; tile += nwarps) {
    V4 cur[U][C];
    uint64_t ii[U], nxt[U];
    uint32_t lo[U], hi[U];
    bool inb[U], ok[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t i = ii[u] = tile * U + u;
      inb[u] = i < a.n;
      const int64_t r = inb[u] ? __ldg(a.idx + i) : 0;
      ok[u] = inb[u] && (uint64_t)r < a.rows;
      const uint64_t s = a.tbase + (ok[u] ? (uint64_t)r : 0ull) * a.rb;
      lo[u] = 0;
      hi[u] = (uint32_t)a.rb;
      nxt[u] = 0;
      if (ok[u]) {
        if ((s & 127) && r > 0 && hs.find((uint64_t)r) == (uint32_t)(i + 1) && hs.find((uint64_t)r - 1) != 0u)
          lo[u] = 128u - (uint32_t)(s & 127);
        const uint64_t e = s + a.rb;
        if ((e & 127) && (uint64_t)r + 1 < a.rows) {
          const uint32_t nx = hs.find((uint64_t)r + 1);
          if (nx) {
            hi[u] = (uint32_t)a.rb + 128u - (uint32_t)(e & 127);
            nxt[u] = nx;
          }
        }
      }
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t b = 16u * (uint32_t)(lane + 32 * c);
        cur[u][c] = (ok[u] && b >= lo[u] && b < hi[u]) ? ld_table16(s + b) : v4_zero();
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!inb[u]) continue;
      const uint64_t d = a.out + ii[u] * a.rb;
#pragma unroll
      for (int c = 0; c < C; ++c) {
        const uint32_t b = 16u * (uint32_t)(lane + 32 * c);
        if (b < lo[u] || b >= hi[u]) continue;
        if (b < a.rb) st16(d + b, cur[u][c]);
        else st16(a.out + (nxt[u] - 1) * a.rb + (b - a.rb), cur[u][c]);
      }
      if (!ok[u] && lane == 0) record_bad(a, ii[u]);
    }
  }
}

}  // namespace ut
