// ut_sample.cu — GPU-side multi-hop neighbour sampling over a host-resident CSR graph
// (SURVEY NEXT-2), the step before the gather that the paper leaves to the CPU ("CPUs need to
// generate subgraphs for each mini-batch and constantly traverse input graphs to identify
// neighboring nodes"; "44%-99%" of training time). The CSR stays in host
// memory and is read by GPU threads through its device mapping, like the feature table.
//
// Semantics are DESIGN.md reading R17 (identical to oracle/ut_oracle_sample.c, which is written
// independently): frontier_0 = seeds (first-appearance unique); at hop h every frontier node v
// takes min(deg, f_h) neighbour slots — all of them when deg <= f_h, else one per stratum
// [floor(t*deg/f), floor((t+1)*deg/f)) picked by the counter hash H(seed, h, v, t); the new
// frontier is the old one followed by the not-yet-seen candidates in (v, t) order.
//
// Per hop: k_count (degree, slot count per frontier node) -> exclusive scan -> k_sample (one
// thread per sample, binary search for its frontier node, one 4-B read of `indices` over the
// link) -> first-appearance dedup with an epoch-tagged per-node atomicMin table (k_first,
// k_keep) -> scan of the keep flags -> k_append. Two host syncs per hop read the sizes.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <new>

#include "ut.h"
#include "ut_internal.h"

using namespace utx;

namespace {

constexpr uint64_t kPhi = 0x9E3779B97F4A7C15ull;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  uint64_t z = x + kPhi;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// H(seed, hop, v, t) of reading R17.
__device__ __forceinline__ uint64_t sample_hash(uint64_t seed, uint64_t hop, uint64_t v, uint64_t t) {
  return mix64(mix64(mix64(seed + (hop + 1) * kPhi) ^ v) + t);
}

__global__ void k_count(const int64_t* __restrict__ front, uint64_t nf, const int64_t* indptr,
                        uint32_t fanout, uint64_t* __restrict__ base, uint64_t* __restrict__ deg,
                        uint32_t* __restrict__ cnt) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nf) return;
  const int64_t v = front[i];
  const int64_t b = indptr[v], e = indptr[v + 1];
  const uint64_t d = (uint64_t)(e - b);
  base[i] = (uint64_t)b;
  deg[i] = d;
  cnt[i] = (uint32_t)(d < fanout ? d : fanout);
}

__global__ void k_sample(const int64_t* __restrict__ front, uint64_t nf, const uint64_t* __restrict__ base,
                         const uint64_t* __restrict__ deg, const uint32_t* __restrict__ off,
                         uint64_t total, uint32_t fanout, uint64_t seed, uint32_t hop,
                         const int32_t* indices, int64_t* __restrict__ cand) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= total) return;
  // frontier node of sample j: the last i with off[i] <= j
  uint64_t lo = 0, hi = nf;
  while (hi - lo > 1) {
    const uint64_t mid = (lo + hi) >> 1;
    if (off[mid] <= j) lo = mid;
    else hi = mid;
  }
  const uint64_t t = j - off[lo];
  const uint64_t d = deg[lo];
  uint64_t slot = t;
  if (d > fanout) {
    const uint64_t s0 = t * d / fanout, s1 = (t + 1) * d / fanout;
    slot = s0 + sample_hash(seed, hop, (uint64_t)front[lo], t) % (s1 - s0);
  }
  cand[j] = (int64_t)indices[base[lo] + slot];
}

// First-appearance dedup against the frontier: firstpos[c] keeps the smallest candidate
// position of node c in this round, tagged with the round's epoch in the high word (a newer
// round's tag is always smaller, so the table is never cleared).
__global__ void k_first(const int64_t* __restrict__ cand, uint64_t m, uint64_t n_nodes,
                        const uint8_t* __restrict__ in_front, unsigned long long* firstpos,
                        uint64_t tag_hi, unsigned long long* err) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint64_t c = (uint64_t)cand[j];
  if (c >= n_nodes) {
    atomicMin(err, (unsigned long long)j);
    return;
  }
  if (!in_front[c]) atomicMin(firstpos + c, (unsigned long long)(tag_hi | j));
}

__global__ void k_keep(const int64_t* __restrict__ cand, uint64_t m, uint64_t n_nodes,
                       const uint8_t* __restrict__ in_front, const unsigned long long* __restrict__ firstpos,
                       uint64_t tag_hi, uint32_t* __restrict__ keep) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const uint64_t c = (uint64_t)cand[j];
  keep[j] = (c < n_nodes && !in_front[c] && firstpos[c] == (tag_hi | j)) ? 1u : 0u;
}

__global__ void k_append(const int64_t* __restrict__ cand, uint64_t m, const uint32_t* __restrict__ keep,
                         const uint32_t* __restrict__ pos, int64_t* __restrict__ front, uint64_t nf,
                         uint8_t* __restrict__ in_front) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m || !keep[j]) return;
  const int64_t c = cand[j];
  front[nf + pos[j]] = c;
  in_front[c] = 1;
}

__global__ void k_clear(const int64_t* __restrict__ front, uint64_t nf, uint8_t* __restrict__ in_front) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nf) in_front[front[i]] = 0;
}

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

__global__ void __launch_bounds__(kScanBlock) k_scan_tiles(const uint32_t* __restrict__ in, uint64_t m,
                                                         uint32_t* __restrict__ out,
                                                         uint32_t* __restrict__ tile_sums) {
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
__global__ void __launch_bounds__(kScanBlock) k_scan_sums(uint32_t* sums, uint64_t ntiles,
                                                        uint64_t* total) {
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

__global__ void k_scan_add(uint32_t* out, uint64_t m, const uint32_t* __restrict__ sums) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < m) out[i] += sums[i / kScanTile];
}

inline int blocks_for(uint64_t n, int per = 256) { return (int)std::max<uint64_t>(1, (n + per - 1) / per); }

}  // namespace

struct ut_graph {
  const int64_t* indptr = nullptr;
  const int32_t* indices = nullptr;
  uint64_t n_nodes = 0, n_edges = 0;
  Pin ip_pin, ix_pin;
  int indptr_hbm = 0;                    // ut_graph_set_option("indptr=hbm")
  std::mutex mu;
  struct Dev {
    bool init = false;
    uint64_t indptr_dev = 0, indices_dev = 0;
    int64_t* indptr_copy = nullptr;      // HBM copy when indptr_hbm
    uint8_t* in_front = nullptr;         // n_nodes flags, all zero between calls
    unsigned long long* firstpos = nullptr;   // n_nodes epoch-tagged positions
    unsigned long long* err = nullptr;
    uint64_t* total_dev = nullptr;       // scan totals
    uint64_t* total_host = nullptr;      // pinned mirror
    uint32_t epoch = 0;
    cudaMemPool_t pool = nullptr;
  } dev[64];
};

namespace {

int graph_dev(ut_graph* g, ut_graph::Dev** out) {
  int d = 0;
  cudaError_t e = cudaGetDevice(&d);
  if (e != cudaSuccess) return cuda_err(e, "cudaGetDevice");
  if (d < 0 || d >= 64) return set_err(UT_ENOTSUP, "device %d", d);
  ut_graph::Dev* s = &g->dev[d];
  if (!s->init) {
    if (pin_device_ptr(g->ip_pin, g->indptr, &s->indptr_dev) != UT_OK) return UT_ECUDA;
    if (pin_device_ptr(g->ix_pin, g->indices, &s->indices_dev) != UT_OK) return UT_ECUDA;
    const uint64_t n = std::max<uint64_t>(1, g->n_nodes);
    if ((e = cudaMalloc(&s->in_front, n)) != cudaSuccess ||
        (e = cudaMalloc(&s->firstpos, n * sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMalloc(&s->err, sizeof(unsigned long long))) != cudaSuccess ||
        (e = cudaMalloc(&s->total_dev, 2 * sizeof(uint64_t))) != cudaSuccess ||
        (e = cudaMallocHost(&s->total_host, 2 * sizeof(uint64_t))) != cudaSuccess) {
      cudaGetLastError();
      return set_err(UT_ENOMEM, "sampler state for %llu nodes", (unsigned long long)n);
    }
    cudaMemset(s->in_front, 0, n);
    cudaMemset(s->firstpos, 0xff, n * sizeof(unsigned long long));
    cudaMemset(s->err, 0xff, sizeof(unsigned long long));
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = d;
    if ((e = cudaMemPoolCreate(&s->pool, &props)) != cudaSuccess) return cuda_err(e, "cudaMemPoolCreate");
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(s->pool, cudaMemPoolAttrReleaseThreshold, &keep);
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return cuda_err(e, "sampler init");
    s->init = true;
  }
  if (g->indptr_hbm && !s->indptr_copy) {
    const uint64_t bytes = (g->n_nodes + 1) * sizeof(int64_t);
    if ((e = cudaMalloc(&s->indptr_copy, bytes)) != cudaSuccess) {
      cudaGetLastError();
      return set_err(UT_ENOMEM, "HBM copy of indptr");
    }
    if ((e = cudaMemcpy(s->indptr_copy, g->indptr, bytes, cudaMemcpyHostToDevice)) != cudaSuccess)
      return cuda_err(e, "indptr H2D");
  }
  *out = s;
  return UT_OK;
}

// exclusive scan of in[0..m) into out, grand total into *total_dev (device)
cudaError_t scan_u32(const uint32_t* in, uint32_t* out, uint64_t m, uint64_t* total_dev,
                     uint32_t* tile_sums, cudaStream_t st) {
  const uint64_t ntiles = (m + kScanTile - 1) / kScanTile;
  if (m) k_scan_tiles<<<(int)ntiles, kScanBlock, 0, st>>>(in, m, out, tile_sums);
  k_scan_sums<<<1, kScanBlock, 0, st>>>(tile_sums, ntiles, total_dev);
  if (m > kScanTile) k_scan_add<<<blocks_for(m), 256, 0, st>>>(out, m, tile_sums);
  return cudaGetLastError();
}

int read_total(ut_graph::Dev* s, cudaStream_t st, uint64_t* v) {
  cudaError_t e = cudaMemcpyAsync(s->total_host, s->total_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) return cuda_err(e, "sampler size read-back");
  *v = s->total_host[0];
  return UT_OK;
}

template <typename T>
int pool_alloc(ut_graph::Dev* s, T** p, uint64_t count, cudaStream_t st) {
  cudaError_t e = cudaMallocFromPoolAsync((void**)p, std::max<uint64_t>(1, count) * sizeof(T), s->pool, st);
  if (e != cudaSuccess) return cuda_err(e, "cudaMallocFromPoolAsync(sampler)");
  return UT_OK;
}

}  // namespace

extern "C" {

ut_graph* ut_graph_register(const int64_t* indptr, const int32_t* indices, uint64_t n_nodes,
                            uint64_t n_edges) {
  if (!indptr || (!indices && n_edges)) return set_err(UT_EINVAL, "NULL CSR array"), nullptr;
  if (n_nodes == 0 || n_nodes >= (1ull << 31)) return set_err(UT_EINVAL, "n_nodes must be in [1, 2^31)"), nullptr;
  if ((uint64_t)indptr[n_nodes] != n_edges || indptr[0] != 0)
    return set_err(UT_EINVAL, "indptr[0] must be 0 and indptr[n_nodes] == n_edges"), nullptr;
  ut_graph* g = new (std::nothrow) ut_graph;
  if (!g) return set_err(UT_ENOMEM, "out of host memory"), nullptr;
  g->indptr = indptr;
  g->indices = indices;
  g->n_nodes = n_nodes;
  g->n_edges = n_edges;
  static const int32_t dummy = 0;
  if (pin_host(indptr, (n_nodes + 1) * sizeof(int64_t), true, &g->ip_pin) != UT_OK ||
      pin_host(n_edges ? (const void*)indices : (const void*)&dummy,
               std::max<uint64_t>(1, n_edges) * sizeof(int32_t), true, &g->ix_pin) != UT_OK) {
    unpin_host(&g->ip_pin);
    delete g;
    return nullptr;
  }
  if (!n_edges) g->indices = &dummy;
  ut_graph::Dev* s;
  if (graph_dev(g, &s) != UT_OK) {
    ut_graph_release(g);
    return nullptr;
  }
  return g;
}

int ut_graph_release(ut_graph* g) {
  if (!g) return UT_OK;
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < 64; ++d) {
    ut_graph::Dev& s = g->dev[d];
    if (!s.init && !s.indptr_copy) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    cudaFree(s.in_front);
    cudaFree(s.firstpos);
    cudaFree(s.err);
    cudaFree(s.total_dev);
    cudaFreeHost(s.total_host);
    cudaFree(s.indptr_copy);
    if (s.pool) cudaMemPoolDestroy(s.pool);
  }
  cudaSetDevice(cur);
  unpin_host(&g->ip_pin);
  unpin_host(&g->ix_pin);
  delete g;
  return UT_OK;
}

int ut_graph_set_option(ut_graph* g, const char* opt) {
  if (!g || !opt) return set_err(UT_EINVAL, "NULL argument");
  if (!strcmp(opt, "indptr=hbm")) g->indptr_hbm = 1;
  else if (!strcmp(opt, "indptr=host")) g->indptr_hbm = 0;
  else return set_err(UT_EINVAL, "unknown option '%s'", opt);
  return UT_OK;
}

int ut_sample(ut_graph* g, const int64_t* seeds_dev, uint64_t n_seeds, const int32_t* fanouts,
              int n_hops, uint64_t seed, int64_t* nodes_dev, uint64_t cap, uint64_t* n_out,
              ut_stream_t stream) {
  if (!g || !n_out || (n_seeds && !seeds_dev) || (n_hops > 0 && !fanouts) || n_hops < 0)
    return set_err(UT_EINVAL, "NULL or negative argument");
  for (int h = 0; h < n_hops; ++h)
    if (fanouts[h] < 0) return set_err(UT_EINVAL, "fanout %d is negative", h);
  *n_out = 0;
  if (n_seeds == 0) return UT_OK;
  std::lock_guard<std::mutex> lk(g->mu);
  ut_graph::Dev* s;
  int rc = graph_dev(g, &s);
  if (rc != UT_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t* indptr = g->indptr_hbm ? s->indptr_copy : (const int64_t*)s->indptr_dev;
  const int32_t* indices = (const int32_t*)s->indices_dev;

  // capacity of the frontier: every hop can add at most fanout new nodes per frontier node
  uint64_t fcap = n_seeds;
  for (int h = 0; h < n_hops; ++h) {
    fcap = std::min<uint64_t>(g->n_nodes, fcap + fcap * (uint64_t)fanouts[h]);
  }
  fcap = std::max<uint64_t>(fcap, n_seeds);
  int64_t* front = nullptr;
  if ((rc = pool_alloc(s, &front, fcap, st)) != UT_OK) return rc;
  uint64_t nf = 0;
  int status = UT_OK;
  cudaError_t e = cudaSuccess;

  // merge `m` candidates into the frontier (first appearance, not yet present)
  auto merge = [&](const int64_t* cand, uint64_t m) -> int {
    if (m == 0) return UT_OK;
    if (++s->epoch == 0xFFFFFFFFu) {   // tags exhausted: reset the table once per 4G rounds
      cudaMemsetAsync(s->firstpos, 0xff, g->n_nodes * sizeof(unsigned long long), st);
      s->epoch = 1;
    }
    const uint64_t tag_hi = (uint64_t)(0xFFFFFFFFu - s->epoch) << 32;
    uint32_t *keep = nullptr, *pos = nullptr, *sums = nullptr;
    int r;
    if ((r = pool_alloc(s, &keep, m, st)) != UT_OK || (r = pool_alloc(s, &pos, m, st)) != UT_OK ||
        (r = pool_alloc(s, &sums, m / kScanTile + 1, st)) != UT_OK)
      return r;
    k_first<<<blocks_for(m), 256, 0, st>>>(cand, m, g->n_nodes, s->in_front, s->firstpos, tag_hi, s->err);
    k_keep<<<blocks_for(m), 256, 0, st>>>(cand, m, g->n_nodes, s->in_front, s->firstpos, tag_hi, keep);
    if ((e = scan_u32(keep, pos, m, s->total_dev, sums, st)) != cudaSuccess) return cuda_err(e, "scan");
    k_append<<<blocks_for(m), 256, 0, st>>>(cand, m, keep, pos, front, nf, s->in_front);
    uint64_t added = 0;
    if ((r = read_total(s, st, &added)) != UT_OK) return r;
    nf += added;
    cudaFreeAsync(keep, st);
    cudaFreeAsync(pos, st);
    cudaFreeAsync(sums, st);
    return UT_OK;
  };

  status = merge(seeds_dev, n_seeds);
  unsigned long long bad = ~0ull;
  if (status == UT_OK) {
    cudaMemcpyAsync(&s->total_host[1], s->err, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    bad = s->total_host[1];
    if (bad != ~0ull) {
      cudaMemsetAsync(s->err, 0xff, sizeof(unsigned long long), st);
      status = set_err(UT_ERANGE, "seed %llu is out of range", bad);
    }
  }
  for (int h = 0; h < n_hops && status == UT_OK; ++h) {
    const uint32_t f = (uint32_t)fanouts[h];
    if (f == 0 || nf == 0) continue;
    uint64_t *base = nullptr, *deg = nullptr;
    uint32_t *cnt = nullptr, *off = nullptr, *sums = nullptr;
    int64_t* cand = nullptr;
    if ((status = pool_alloc(s, &base, nf, st)) != UT_OK || (status = pool_alloc(s, &deg, nf, st)) != UT_OK ||
        (status = pool_alloc(s, &cnt, nf, st)) != UT_OK || (status = pool_alloc(s, &off, nf, st)) != UT_OK ||
        (status = pool_alloc(s, &sums, nf / kScanTile + 1, st)) != UT_OK)
      break;
    k_count<<<blocks_for(nf), 256, 0, st>>>(front, nf, indptr, f, base, deg, cnt);
    if ((e = scan_u32(cnt, off, nf, s->total_dev, sums, st)) != cudaSuccess) {
      status = cuda_err(e, "scan");
      break;
    }
    uint64_t total = 0;
    if ((status = read_total(s, st, &total)) != UT_OK) break;
    if ((status = pool_alloc(s, &cand, total, st)) != UT_OK) break;
    if (total)
      k_sample<<<blocks_for(total), 256, 0, st>>>(front, nf, base, deg, off, total, f, seed,
                                                  (uint32_t)h, indices, cand);
    if ((e = cudaGetLastError()) != cudaSuccess) {
      status = cuda_err(e, "k_sample");
      break;
    }
    status = merge(cand, total);
    cudaFreeAsync(base, st);
    cudaFreeAsync(deg, st);
    cudaFreeAsync(cnt, st);
    cudaFreeAsync(off, st);
    cudaFreeAsync(sums, st);
    cudaFreeAsync(cand, st);
  }
  if (status == UT_OK) {
    *n_out = nf;
    if (nf > cap || !nodes_dev) status = set_err(UT_EINVAL, "nodes buffer holds %llu, need %llu",
                                                 (unsigned long long)cap, (unsigned long long)nf);
    else if ((e = cudaMemcpyAsync(nodes_dev, front, nf * sizeof(int64_t), cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
      status = cuda_err(e, "copy nodes");
  }
  if (nf) k_clear<<<blocks_for(nf), 256, 0, st>>>(front, nf, s->in_front);
  cudaFreeAsync(front, st);
  if ((e = cudaGetLastError()) != cudaSuccess && status == UT_OK) status = cuda_err(e, "sampler");
  return status;
}

}  // extern "C"
