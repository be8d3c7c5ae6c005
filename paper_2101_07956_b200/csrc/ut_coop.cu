// ut_coop.cu — cooperative multi-rank gather over peer device memory.
//
// The paper's path has every GPU pull its own minibatch's rows over its own host link
// (Fig. 2b). When several GPUs of a box gather from one shared host table in
// the same step, their minibatches overlap (hub nodes are sampled by everyone: products-shaped
// minibatches of 8 ranks share 53 % of their rows) and the host side — the links
// behind a shared PCIe switch, host DRAM — moves the shared rows once per rank. Here the ranks
// split the table into row blocks owned round-robin, and one step is
//
//   dispatch  each rank sends every index to the owner of its row block: warp-aggregated slot
//             reservation, then P2P stores of the row id into the owner's inbox (NVLink peer
//             memory; on one GPU shared by several processes, CUDA IPC memory of that GPU);
//   fetch     each owner deduplicates the requests of all ranks (epoch-tagged atomicMax table,
//             the first request of a row wins) and gathers its unique rows ONCE from host memory
//             with the ordinary unified-tensor gather (ut_gather_dn: plans, reorder, shapes)
//             into its staging rows;
//   combine   each rank copies its rows out of the owners' staging rows (P2P loads) into
//             out[i] in its own index order.
//
// Result: out[i] = table row idx[i], byte for byte — the same definition as ut_gather
// (oracle/ut_oracle.c); out-of-range indices are zero-filled and their first
// position recorded (reading R4). Host bytes per step fall from sum(n_r)*rb to |union|*rb.
//
// Synchronisation between the phases is either the caller's host barrier (ut_coop_dispatch /
// ut_coop_fetch / ut_coop_combine with stream syncs and a process-group barrier between them) or
// device-side (ut_coop_gather): every rank writes the step's epoch into a flag word of every peer
// and its stream waits for all peers' flags (cuStreamWriteValue32 / cuStreamWaitValue32, no SM
// spins and no host round trip). The symmetric regions are double-buffered by step parity, so
// step k+1's dispatch never overwrites what a slow peer still reads for step k.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <new>
#include <vector>

#include "ut.h"
#include "ut_internal.h"

using namespace utx;

namespace {

constexpr int kMaxWorld = 64;
constexpr uint32_t kFull = 0xffffffffu;

// Row-block ownership: block b = id / R is owned by rank b mod world; within the owner, the
// block's rows have the dense local index (b / world) * R + id mod R.
struct Owner {
  uint64_t R;
  uint32_t world;
  __host__ __device__ uint32_t of(uint64_t id) const { return (uint32_t)((id / R) % world); }
  __host__ __device__ uint64_t local(uint64_t id) const { return (id / R / world) * R + id % R; }
};

// Row-block size: 2 MiB of rows (one translation region), shrunk so the table has at least
// 64 blocks per rank (load balance on small tables), at least one row.
uint64_t block_rows(uint64_t rows, uint64_t rb, int world) {
  uint64_t R = std::max<uint64_t>(1, (2ull << 20) / rb);
  const uint64_t want = 64ull * (uint64_t)world;
  if ((rows + R - 1) / R < want) R = std::max<uint64_t>(1, rows / want);
  return R;
}

// Layout of one parity half of the symmetric region (identical on every rank).
struct Layout {
  uint64_t count, inbox, slot, stage, half;   // byte offsets inside a half, half size
  uint64_t flags;                             // offset of the flag words (after both halves)
  uint64_t total;
};

uint64_t up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

Layout layout_for(int world, uint64_t cap, uint64_t rb) {
  Layout L{};
  const uint64_t W = (uint64_t)world;
  L.count = 0;
  L.inbox = up(W * 8, 256);
  L.slot = up(L.inbox + W * cap * 8, 256);
  L.stage = up(L.slot + W * cap * 4, 256);
  L.half = up(L.stage + W * cap * rb, 256);
  L.flags = 2 * L.half;
  L.total = L.flags + up(2 * W * 4, 256);     // flags[barrier 0/1][source rank]
  return L;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// ---- dispatch -----------------------------------------------------------------------------
// Every index goes to its owner: lanes of a warp with the same owner reserve consecutive inbox
// slots with one atomicAdd (__match_any_sync groups them), then store the row id into the
// owner's inbox row for this rank. map[i] = (owner << 32) | slot, or ~0 for a bad index.
__global__ void k_dispatch(const int64_t* __restrict__ idx, uint64_t n, uint64_t rows, Owner own,
                           uint8_t* const* __restrict__ peers, uint64_t parity_off, uint64_t inbox_off,
                           uint64_t cap, uint32_t rank, uint32_t* __restrict__ cnt,
                           uint64_t* __restrict__ map, unsigned long long* __restrict__ err) {
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  for (uint64_t base = w * 32; base < n; base += warps * 32) {
    const uint64_t i = base + lane;
    const bool active = i < n;
    const int64_t id = active ? idx[i] : 0;
    const bool valid = active && id >= 0 && (uint64_t)id < rows;
    if (active && !valid) {
      atomicMin(err, (unsigned long long)i);
      map[i] = ~0ull;
    }
    const int o = valid ? (int)own.of((uint64_t)id) : -1;
    const uint32_t grp = __match_any_sync(kFull, o);
    const int leader = __ffs(grp) - 1;
    uint32_t b = 0;
    if (valid && (int)lane == leader) b = atomicAdd(&cnt[o], (uint32_t)__popc(grp));
    b = __shfl_sync(kFull, b, valid ? leader : (int)lane);
    if (valid) {
      const uint32_t slot = b + (uint32_t)__popc(grp & ((1u << lane) - 1));
      int64_t* inbox = (int64_t*)(peers[o] + parity_off + inbox_off) + (uint64_t)rank * cap;
      inbox[slot] = id;
      map[i] = ((uint64_t)o << 32) | slot;
    }
  }
}

// count[rank] in every owner's region = the number of requests this rank sent it.
__global__ void k_publish(uint8_t* const* __restrict__ peers, uint64_t parity_off, uint32_t rank,
                          uint32_t world, const uint32_t* __restrict__ cnt) {
  const uint32_t o = threadIdx.x;
  if (o < world) ((uint64_t*)(peers[o] + parity_off))[rank] = cnt[o];
}

// ---- fetch (owner side) -------------------------------------------------------------------
// Requests are addressed e = src * cap + slot. Pass 1: per row, the smallest e of this epoch
// wins (atomicMax of (epoch << 32) | ~e; older epochs compare smaller, so the table is never
// cleared). Pass 2: winners take a unique staging slot and list their row for the host gather.
// Pass 3: every request learns its row's staging slot.
struct FetchArgs {
  const uint64_t* count;     // [world] requests per source (own region, this parity)
  const int64_t* inbox;      // [world][cap]
  uint32_t* slot_of;         // [world][cap] staging slot of each request (read by requesters)
  unsigned long long* tag;   // [local rows] epoch-tagged winner
  uint32_t* wslot;           // [world][cap] staging slot of each winning request
  int64_t* uniq;             // [world*cap] rows to fetch from the host
  unsigned long long* u;     // [0] unique rows this step, [1] all-time unique, [2] all-time requests
  uint64_t cap;
  uint32_t world;
  uint32_t epoch;
  Owner own;
  bool partitioned;          // the fetch reads a per-rank partition at the row's local index
};

template <int PASS>
__global__ void k_dedup(FetchArgs f) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t total = f.cap * f.world;
  for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x; base < total; base += stride) {
    const uint64_t e = base + threadIdx.x;
    bool live = false;
    uint64_t l = 0;
    int64_t id = 0;
    if (e < total) {
      const uint64_t src = e / f.cap, slot = e - src * f.cap;
      live = slot < f.count[src];
      if (live) {
        id = f.inbox[e];
        l = f.own.local((uint64_t)id);
      }
    }
    if (PASS == 1) {
      if (live) atomicMax(&f.tag[l], ((unsigned long long)f.epoch << 32) | (uint32_t)~(uint32_t)e);
    } else if (PASS == 2) {
      // winners take consecutive staging slots: one atomicAdd per block and loop iteration
      __shared__ uint32_t warp_tot[32];
      __shared__ unsigned long long block_base;
      const bool win = live && (uint32_t)~(uint32_t)f.tag[l] == (uint32_t)e;
      const uint32_t wm = __ballot_sync(kFull, win);
      const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
      if (lane == 0) warp_tot[warp] = __popc(wm);
      __syncthreads();
      if (threadIdx.x == 0) {
        uint32_t tot = 0;
        for (uint32_t k = 0; k < nw; ++k) {
          const uint32_t c = warp_tot[k];
          warp_tot[k] = tot;                 // exclusive prefix over the block's warps
          tot += c;
        }
        block_base = tot ? atomicAdd(&f.u[0], (unsigned long long)tot) : 0ull;
      }
      __syncthreads();
      if (win) {
        const uint64_t s = block_base + warp_tot[warp] + __popc(wm & ((1u << lane) - 1));
        f.uniq[s] = f.partitioned ? (int64_t)l : id;
        f.wslot[e] = (uint32_t)s;
      }
      __syncthreads();                       // warp_tot / block_base reused next iteration
    } else {
      if (live) f.slot_of[e] = f.wslot[~(uint32_t)f.tag[l]];
    }
  }
}

// all-time counters: unique rows fetched, requests received (sum of the sources' counts)
__global__ void k_unique_total(unsigned long long* u, const uint64_t* count, uint32_t world) {
  uint64_t req = 0;
  for (uint32_t q = 0; q < world; ++q) req += count[q];
  u[1] += u[0];
  u[2] += req;
}

// ---- combine (requester side) ---------------------------------------------------------------
// out[i] = staging row slot_of[rank][slot] of owner o, copied with W-byte words (W = the widest
// width that rb, the staging rows and out all allow); a warp per row, two rows in flight.
template <typename T>
__global__ void k_combine(const uint64_t* __restrict__ map, uint64_t n, uint64_t rb,
                          uint8_t* const* __restrict__ peers, uint64_t parity_off, uint64_t slot_off,
                          uint64_t stage_off, uint64_t cap, uint32_t rank, uint8_t* __restrict__ out) {
  const uint64_t warps = (uint64_t)gridDim.x * (blockDim.x >> 5);
  const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = lane_id();
  const uint64_t words = rb / sizeof(T);
  for (uint64_t i0 = w * 2; i0 < n; i0 += warps * 2) {
    const T* src[2] = {nullptr, nullptr};
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const uint64_t i = i0 + k;
      if (i >= n) continue;
      const uint64_t m = map[i];
      if (m == ~0ull) continue;
      const uint32_t o = (uint32_t)(m >> 32), slot = (uint32_t)m;
      const uint8_t* reg = peers[o] + parity_off;
      const uint32_t s = ((const uint32_t*)(reg + slot_off))[(uint64_t)rank * cap + slot];
      src[k] = (const T*)(reg + stage_off + (uint64_t)s * rb);
    }
    for (uint64_t j = lane; j < words; j += 64) {
      T v[2][2];
#pragma unroll
      for (int k = 0; k < 2; ++k)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint64_t jj = j + 32 * h;
          v[k][h] = (src[k] && jj < words) ? src[k][jj] : T{};
        }
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        if (i0 + k >= n) continue;
        T* d = (T*)(out + (i0 + k) * rb);
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (j + 32 * h < words) d[j + 32 * h] = v[k][h];
      }
    }
  }
}

struct alignas(16) W16 {
  uint4 v;
};

typedef CUresult (*PWrite)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
typedef CUresult (*PWait)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

template <typename F>
F drv(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q{};
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &q) != cudaSuccess ||
      q != cudaDriverEntryPointSuccess)
    return nullptr;
  return reinterpret_cast<F>(fn);
}

}  // namespace

struct ut_coop {
  const ut_table* t = nullptr;
  int world = 1, rank = 0, dev = 0, sms = 148;
  uint64_t cap = 0, rows = 0, rb = 0;
  Owner own{1, 1};
  Layout L{};
  uint8_t* region = nullptr;                 // own symmetric region (cudaMalloc, IPC-exportable)
  uint8_t* peer_host[kMaxWorld] = {};        // every rank's region in this process (own = region)
  bool opened[kMaxWorld] = {};
  uint8_t** peers_dev = nullptr;             // device copy of peer_host
  unsigned long long* tag = nullptr;
  uint64_t tag_len = 0;
  uint32_t* wslot = nullptr;
  int64_t* uniq = nullptr;
  unsigned long long* u = nullptr;           // [0] step unique, [1] total unique, [2] total requests
  uint64_t* map = nullptr;
  uint32_t* cnt = nullptr;
  unsigned long long* err = nullptr;
  uint32_t epoch = 0;                        // steps dispatched so far
  bool partitioned = false;                  // t holds only this rank's rows, in local order
  uint64_t last_n = 0;
  uint64_t steps = 0, requested = 0, launches = 0, memops = 0;
  PWrite write32 = nullptr;
  PWait wait32 = nullptr;
};

namespace {

uint64_t parity_off(const ut_coop* c) { return (uint64_t)(c->epoch & 1) * c->L.half; }

int grid(const ut_coop* c, uint64_t threads) {
  return (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)c->sms * 8, (threads + 255) / 256));
}

// Device-side barrier `b` of the current epoch: write the epoch into flags[b][rank] of every
// peer, then wait until every peer has written it into ours.
int device_barrier(ut_coop* c, int b, cudaStream_t st) {
  if (!c->write32 || !c->wait32) return set_err(UT_ENOTSUP, "stream memory operations unavailable");
  for (int q = 0; q < c->world; ++q) {
    CUdeviceptr f = (CUdeviceptr)(c->peer_host[q] + c->L.flags) + (CUdeviceptr)((b * c->world + c->rank) * 4);
    if (c->write32((CUstream)st, f, c->epoch, 0) != CUDA_SUCCESS)
      return set_err(UT_ECUDA, "cuStreamWriteValue32 to rank %d failed", q);
  }
  for (int q = 0; q < c->world; ++q) {
    CUdeviceptr f = (CUdeviceptr)(c->region + c->L.flags) + (CUdeviceptr)((b * c->world + q) * 4);
    if (c->wait32((CUstream)st, f, c->epoch, CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      return set_err(UT_ECUDA, "cuStreamWaitValue32 on rank %d failed", q);
  }
  c->memops += 2 * (uint64_t)c->world;
  return UT_OK;
}

int check_dev(const ut_coop* c) {
  int d = -1;
  cudaGetDevice(&d);
  if (d != c->dev) return set_err(UT_EINVAL, "current device %d is not the coop's device %d", d, c->dev);
  for (int q = 0; q < c->world; ++q)
    if (!c->peer_host[q]) return set_err(UT_EINVAL, "peer regions not opened (ut_coop_open)");
  return UT_OK;
}

}  // namespace

extern "C" {

static ut_coop* coop_create(const ut_table* t, uint64_t full_rows, bool partitioned, int world,
                            int rank, uint64_t max_n) {
  if (!t) return set_err(UT_EINVAL, "table is NULL"), nullptr;
  if (world < 1 || world > kMaxWorld || rank < 0 || rank >= world)
    return set_err(UT_EINVAL, "world %d / rank %d out of range (world <= %d)", world, rank, kMaxWorld), nullptr;
  if (max_n == 0 || max_n * (uint64_t)world >= (1ull << 31))
    return set_err(UT_EINVAL, "max_n must be >= 1 and world*max_n < 2^31"), nullptr;
  ut_table_info info{};
  if (ut_table_get_info(t, &info) != UT_OK) return nullptr;
  ut_coop* c = new (std::nothrow) ut_coop;
  if (!c) return set_err(UT_ENOMEM, "out of host memory"), nullptr;
  c->t = t;
  c->world = world;
  c->rank = rank;
  c->cap = max_n;
  c->rows = partitioned ? full_rows : info.rows;
  c->rb = info.row_bytes;
  c->partitioned = partitioned;
  if (c->rows == 0) {
    delete c;
    return set_err(UT_EINVAL, "rows is 0"), nullptr;
  }
  if (max_n > UINT64_MAX / 4 / c->rb / (uint64_t)world) {
    delete c;
    return set_err(UT_EINVAL, "world*max_n*row_bytes overflows"), nullptr;
  }
  c->own = Owner{block_rows(c->rows, c->rb, world), (uint32_t)world};
  c->L = layout_for(world, max_n, c->rb);
  cudaGetDevice(&c->dev);
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, c->dev);
  const uint64_t nblocks = (c->rows + c->own.R - 1) / c->own.R;
  c->tag_len = ((nblocks + world - 1) / world) * c->own.R;
  if (partitioned && info.rows < c->tag_len) {
    const uint64_t need = c->tag_len;
    delete c;
    return set_err(UT_EINVAL, "partition has %llu rows, this rank's blocks need %llu (ut_coop_partition_ids)",
                   (unsigned long long)info.rows, (unsigned long long)need), nullptr;
  }
  const uint64_t E = (uint64_t)world * max_n;
  cudaError_t e = cudaMalloc(&c->region, c->L.total);
  if (e == cudaSuccess) e = cudaMemset(c->region, 0, c->L.total);
  if (e == cudaSuccess) e = cudaMalloc(&c->peers_dev, sizeof(uint8_t*) * world);
  if (e == cudaSuccess) e = cudaMalloc(&c->tag, c->tag_len * 8);
  if (e == cudaSuccess) e = cudaMemset(c->tag, 0, c->tag_len * 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->wslot, E * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->uniq, E * 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->u, 4 * 8);
  if (e == cudaSuccess) e = cudaMemset(c->u, 0, 4 * 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->map, max_n * 8);
  if (e == cudaSuccess) e = cudaMalloc(&c->cnt, (uint64_t)world * 4);
  if (e == cudaSuccess) e = cudaMalloc(&c->err, 8);
  if (e == cudaSuccess) e = cudaMemset(c->err, 0xff, 8);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);   // memsets landed
  if (e != cudaSuccess) {
    cuda_err(e, "ut_coop_create allocation");
    ut_coop_release(c);
    return nullptr;
  }
  c->peer_host[rank] = c->region;
  c->write32 = drv<PWrite>("cuStreamWriteValue32");
  c->wait32 = drv<PWait>("cuStreamWaitValue32");
  if (world == 1 && ut_coop_open(c, nullptr) != UT_OK) {
    ut_coop_release(c);
    return nullptr;
  }
  return c;
}

ut_coop* ut_coop_create(const ut_table* t, int world, int rank, uint64_t max_n) {
  return coop_create(t, 0, false, world, rank, max_n);
}

ut_coop* ut_coop_create_partitioned(const ut_table* part, uint64_t rows, int world, int rank,
                                    uint64_t max_n) {
  return coop_create(part, rows, true, world, rank, max_n);
}

uint64_t ut_coop_partition_ids(uint64_t rows, uint64_t row_bytes, int world, int rank, int64_t* ids,
                               uint64_t cap) {
  if (rows == 0 || row_bytes == 0 || world < 1 || rank < 0 || rank >= world) return 0;
  const Owner o{block_rows(rows, row_bytes, world), (uint32_t)world};
  const uint64_t nblocks = (rows + o.R - 1) / o.R;
  const uint64_t local_rows = ((nblocks + world - 1) / world) * o.R;
  if (ids && cap >= local_rows) {
    for (uint64_t l = 0; l < local_rows; ++l) {
      const uint64_t b = (l / o.R) * (uint64_t)world + (uint64_t)rank;   // inverse of Owner::local
      const uint64_t id = b * o.R + l % o.R;
      ids[l] = id < rows ? (int64_t)id : -1;
    }
  }
  return local_rows;
}

int ut_coop_export(const ut_coop* c, void* handle_out, uint64_t* region_bytes) {
  if (!c || !handle_out) return set_err(UT_EINVAL, "coop or handle_out is NULL");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, c->region);
  if (e != cudaSuccess) return cuda_err(e, "cudaIpcGetMemHandle");
  static_assert(sizeof(h) == UT_COOP_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof h);
  if (region_bytes) *region_bytes = c->L.total;
  return UT_OK;
}

int ut_coop_open(ut_coop* c, const void* handles) {
  if (!c) return set_err(UT_EINVAL, "coop is NULL");
  if (c->world > 1 && !handles) return set_err(UT_EINVAL, "handles is NULL");
  for (int q = 0; q < c->world; ++q) {
    if (q == c->rank || c->peer_host[q]) continue;
    cudaIpcMemHandle_t h;
    memcpy(&h, (const uint8_t*)handles + (size_t)q * UT_COOP_HANDLE_BYTES, sizeof h);
    void* p = nullptr;
    cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_err(e, "cudaIpcOpenMemHandle");
    c->peer_host[q] = (uint8_t*)p;
    c->opened[q] = true;
  }
  // from pageable memory cudaMemcpy may return before the DMA lands: wait for it, since the
  // first step may run on a non-blocking stream
  cudaError_t e = cudaMemcpy(c->peers_dev, c->peer_host, sizeof(uint8_t*) * c->world, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(peer table)");
  return UT_OK;
}

int ut_coop_open_local(ut_coop* c, ut_coop* const* peers, int world) {
  if (!c || !peers) return set_err(UT_EINVAL, "coop or peers is NULL");
  if (world != c->world) return set_err(UT_EINVAL, "world %d != the coop's %d", world, c->world);
  if (peers[c->rank] != c) return set_err(UT_EINVAL, "peers[%d] is not this rank's handle", c->rank);
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != c->dev) return set_err(UT_EINVAL, "current device %d is not the coop's device %d", cur, c->dev);
  for (int q = 0; q < world; ++q) {
    const ut_coop* p = peers[q];
    if (!p) return set_err(UT_EINVAL, "peers[%d] is NULL", q);
    if (p->world != world || p->rank != q || p->cap != c->cap || p->rows != c->rows ||
        p->rb != c->rb || p->partitioned != c->partitioned || p->L.total != c->L.total)
      return set_err(UT_EINVAL, "rank %d disagrees on (world, rank, max_n, rows, row_bytes, form)", q);
  }
  for (int q = 0; q < world; ++q) {
    if (q == c->rank) continue;
    const ut_coop* p = peers[q];
    if (p->dev != c->dev) {
      int ok = 0;
      cudaDeviceCanAccessPeer(&ok, c->dev, p->dev);
      if (!ok) return set_err(UT_ENOTSUP, "device %d cannot access device %d (no P2P)", c->dev, p->dev);
      cudaError_t e = cudaDeviceEnablePeerAccess(p->dev, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      else if (e != cudaSuccess) return cuda_err(e, "cudaDeviceEnablePeerAccess");
    }
    c->peer_host[q] = p->region;    // not IPC-opened: ut_coop_release leaves it to its owner
    c->opened[q] = false;
  }
  // from pageable memory cudaMemcpy may return before the DMA lands: wait for it, since the
  // first step may run on a non-blocking stream
  cudaError_t e = cudaMemcpy(c->peers_dev, c->peer_host, sizeof(uint8_t*) * c->world, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaStreamSynchronize(cudaStreamLegacy);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(peer table)");
  // In-process ranks wait for each other on the device (stream memory operations). Loading a
  // kernel lazily (CUDA_MODULE_LOADING=LAZY, the default) while another rank's stream of the
  // same process waits at a barrier can stall both, so every kernel a step launches is loaded
  // now: the coop kernels by their attributes, the host fetch's gather plan (and its reorder
  // stage, when the policy takes it) by one device-count gather of zero rows at the step's size.
  const void* ks[] = {(const void*)k_dispatch, (const void*)k_publish, (const void*)k_dedup<1>,
                      (const void*)k_dedup<2>, (const void*)k_dedup<3>, (const void*)k_unique_total,
                      (const void*)k_combine<W16>, (const void*)k_combine<uint64_t>,
                      (const void*)k_combine<uint32_t>, (const void*)k_combine<uint16_t>,
                      (const void*)k_combine<uint8_t>};
  for (const void* k : ks) {
    cudaFuncAttributes fa;
    if ((e = cudaFuncGetAttributes(&fa, k)) != cudaSuccess) return cuda_err(e, "cudaFuncGetAttributes");
  }
  if ((e = cudaMemsetAsync(c->u, 0, 8, 0)) != cudaSuccess) return cuda_err(e, "cudaMemsetAsync(preload)");
  const int rc = ut_gather_dn(c->t, c->uniq, (const uint64_t*)c->u, c->cap * (uint64_t)c->world,
                              c->region + c->L.stage, nullptr);
  if (rc != UT_OK) return rc;
  if ((e = cudaStreamSynchronize(0)) != cudaSuccess) return cuda_err(e, "preload gather");
  return UT_OK;
}

int ut_coop_dispatch(ut_coop* c, const int64_t* idx_dev, uint64_t n, ut_stream_t stream) {
  if (!c) return set_err(UT_EINVAL, "coop is NULL");
  if (n > c->cap) return set_err(UT_EINVAL, "n = %llu exceeds max_n = %llu", (unsigned long long)n,
                                 (unsigned long long)c->cap);
  if (n > 0 && !idx_dev) return set_err(UT_EINVAL, "idx_dev is NULL");
  int rc = check_dev(c);
  if (rc != UT_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  c->epoch += 1;
  c->last_n = n;
  c->steps += 1;
  c->requested += n;
  const uint64_t po = parity_off(c);
  cudaError_t e = cudaMemsetAsync(c->cnt, 0, (size_t)c->world * 4, st);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemsetAsync(dispatch counters)");
  if (n > 0)
    k_dispatch<<<grid(c, n), 256, 0, st>>>(idx_dev, n, c->rows, c->own, c->peers_dev, po, c->L.inbox,
                                           c->cap, (uint32_t)c->rank, c->cnt, c->map, c->err);
  k_publish<<<1, 64, 0, st>>>(c->peers_dev, po, (uint32_t)c->rank, (uint32_t)c->world, c->cnt);
  c->launches += n > 0 ? 2 : 1;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "coop dispatch");
  return UT_OK;
}

int ut_coop_fetch(ut_coop* c, ut_stream_t stream) {
  if (!c) return set_err(UT_EINVAL, "coop is NULL");
  int rc = check_dev(c);
  if (rc != UT_OK) return rc;
  if (c->epoch == 0) return set_err(UT_EINVAL, "ut_coop_fetch before ut_coop_dispatch");
  cudaStream_t st = (cudaStream_t)stream;
  uint8_t* reg = c->region + parity_off(c);
  FetchArgs f{(const uint64_t*)(reg + c->L.count), (const int64_t*)(reg + c->L.inbox),
              (uint32_t*)(reg + c->L.slot), c->tag, c->wslot, c->uniq, c->u, c->cap,
              (uint32_t)c->world, c->epoch, c->own, c->partitioned};
  const uint64_t E = c->cap * (uint64_t)c->world;
  cudaError_t e = cudaMemsetAsync(c->u, 0, 8, st);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemsetAsync(unique count)");
  k_dedup<1><<<grid(c, E), 256, 0, st>>>(f);
  k_dedup<2><<<grid(c, E), 256, 0, st>>>(f);
  k_dedup<3><<<grid(c, E), 256, 0, st>>>(f);
  k_unique_total<<<1, 1, 0, st>>>(c->u, f.count, (uint32_t)c->world);
  c->launches += 4;
  e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "coop dedup");
  // the unique rows, once, from host memory: the ordinary unified-tensor gather
  return ut_gather_dn(c->t, c->uniq, (const uint64_t*)c->u, E, reg + c->L.stage, stream);
}

int ut_coop_combine(ut_coop* c, void* out_dev, ut_stream_t stream) {
  if (!c) return set_err(UT_EINVAL, "coop is NULL");
  int rc = check_dev(c);
  if (rc != UT_OK) return rc;
  const uint64_t n = c->last_n;
  if (n == 0) return UT_OK;
  if (!out_dev) return set_err(UT_EINVAL, "out_dev is NULL");
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t po = parity_off(c);
  const uint64_t a = (uint64_t)out_dev | c->rb | (uint64_t)c->region | c->L.stage;
  const int g = grid(c, n * 16);
  uint8_t* out = (uint8_t*)out_dev;
#define UT_COMBINE(T) k_combine<T><<<g, 256, 0, st>>>(c->map, n, c->rb, c->peers_dev, po, c->L.slot, \
                                                      c->L.stage, c->cap, (uint32_t)c->rank, out)
  if ((a & 15) == 0) UT_COMBINE(W16);
  else if ((a & 7) == 0) UT_COMBINE(uint64_t);
  else if ((a & 3) == 0) UT_COMBINE(uint32_t);
  else if ((a & 1) == 0) UT_COMBINE(uint16_t);
  else UT_COMBINE(uint8_t);
#undef UT_COMBINE
  c->launches += 1;
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "coop combine");
  return UT_OK;
}

int ut_coop_gather(ut_coop* c, const int64_t* idx_dev, uint64_t n, void* out_dev, ut_stream_t stream) {
  if (!c) return set_err(UT_EINVAL, "coop is NULL");
  // Bad arguments on one rank must not strand its peers at the device barriers: take part in
  // the step with no rows, then report the error.
  int bad = UT_OK;
  if (n > c->cap) bad = set_err(UT_EINVAL, "n = %llu exceeds max_n = %llu", (unsigned long long)n,
                                (unsigned long long)c->cap);
  else if (n > 0 && (!idx_dev || !out_dev)) bad = set_err(UT_EINVAL, "idx_dev/out_dev is NULL");
  if (bad != UT_OK) n = 0;
  int rc = ut_coop_dispatch(c, idx_dev, n, stream);
  if (rc == UT_OK && c->world > 1) rc = device_barrier(c, 0, (cudaStream_t)stream);
  if (rc == UT_OK) {
    // once barrier 0 is enqueued the peers' streams wait for this rank's barrier-1 flags: write
    // them even when the fetch fails (its error is reported after), or the peers hang
    const int frc = ut_coop_fetch(c, stream);
    char fmsg[512] = "";
    if (frc != UT_OK) ut_last_error(fmsg, sizeof fmsg);
    if (c->world > 1) rc = device_barrier(c, 1, (cudaStream_t)stream);
    if (frc != UT_OK) return set_err(frc, "%s", fmsg);
  }
  if (rc == UT_OK) rc = ut_coop_combine(c, out_dev, stream);
  if (rc == UT_OK && bad != UT_OK) {
    char msg[512];
    ut_last_error(msg, sizeof msg);     // keep the argument error, not a later success
    return set_err(bad, "%s (the step ran with n = 0 so the peers are not stranded)", msg);
  }
  return rc;
}

int ut_coop_get_stats(const ut_coop* c, ut_coop_stats* s) {
  if (!c || !s) return set_err(UT_EINVAL, "coop or stats is NULL");
  unsigned long long u[4];
  cudaError_t e = cudaMemcpy(u, c->u, sizeof u, cudaMemcpyDeviceToHost);
  if (e != cudaSuccess) return cuda_err(e, "cudaMemcpy(coop stats)");
  s->steps = c->steps;
  s->requested_rows = c->requested;
  s->owner_requests = u[2];
  s->unique_rows_fetched = u[1];
  s->last_unique_rows = u[0];
  s->kernel_launches = c->launches;
  s->stream_memops = c->memops;
  s->block_rows = c->own.R;
  s->region_bytes = c->L.total;
  return UT_OK;
}

int ut_coop_error_pos(const ut_coop* c, ut_stream_t stream, int64_t* first_bad) {
  if (!c || !first_bad) return set_err(UT_EINVAL, "coop or first_bad is NULL");
  cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "cudaStreamSynchronize");
  unsigned long long v = 0;
  e = cudaMemcpy(&v, c->err, 8, cudaMemcpyDeviceToHost);
  // cleared on `stream` and waited for, so no later step races the clear
  if (e == cudaSuccess) e = cudaMemsetAsync(c->err, 0xff, 8, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return cuda_err(e, "error word");
  *first_bad = v == ~0ull ? -1 : (int64_t)v;
  return v == ~0ull ? UT_OK : UT_ERANGE;
}

uint32_t ut_coop_owner(uint64_t rows, uint64_t row_bytes, int world, int64_t id, uint64_t* local) {
  if (rows == 0 || row_bytes == 0 || world < 1 || id < 0 || (uint64_t)id >= rows) return UINT32_MAX;
  const Owner o{block_rows(rows, row_bytes, world), (uint32_t)world};
  if (local) *local = o.local((uint64_t)id);
  return o.of((uint64_t)id);
}

int ut_coop_release(ut_coop* c) {
  if (!c) return UT_OK;
  int d = -1;
  cudaGetDevice(&d);
  if (d != c->dev) cudaSetDevice(c->dev);
  cudaDeviceSynchronize();
  for (int q = 0; q < c->world; ++q)
    if (c->opened[q]) cudaIpcCloseMemHandle(c->peer_host[q]);
  cudaFree(c->region);
  cudaFree(c->peers_dev);
  cudaFree(c->tag);
  cudaFree(c->wslot);
  cudaFree(c->uniq);
  cudaFree(c->u);
  cudaFree(c->map);
  cudaFree(c->cnt);
  cudaFree(c->err);
  if (d >= 0 && d != c->dev) cudaSetDevice(d);
  delete c;
  return UT_OK;
}

}  // extern "C"
