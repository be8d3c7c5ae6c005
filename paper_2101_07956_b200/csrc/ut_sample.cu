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
// k_keep) -> scan of the keep flags -> k_append. Sizes stay in device memory and launches are
// sized by worst-case bounds, so a call enqueues with no host synchronisation (ut_sample_async,
// CUDA-graph capturable); ut_sample adds one sync at the end to return the count.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <new>

#include "ut.h"
#include "ut_internal.h"
#include "ut_scan.cuh"

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

// All sizes live in device memory (sz[]), so one call enqueues without host synchronisation
// and can be captured in a CUDA graph; launches are sized by host-side worst-case bounds.
enum { SZ_NF = 0, SZ_TOTAL = 1, SZ_ADDED = 2, SZ_EPOCH = 3, SZ_N = 4 };

__global__ void k_count(const int64_t* __restrict__ front, const uint64_t* sz, const int64_t* indptr,
                        uint32_t fanout, uint64_t* __restrict__ base, uint64_t* __restrict__ deg,
                        uint32_t* __restrict__ cnt) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= sz[SZ_NF]) return;
  const int64_t v = front[i];
  const int64_t b = indptr[v], e = indptr[v + 1];
  const uint64_t d = (uint64_t)(e - b);
  base[i] = (uint64_t)b;
  deg[i] = d;
  cnt[i] = (uint32_t)(d < fanout ? d : fanout);
}

__global__ void k_sample(const int64_t* __restrict__ front, const uint64_t* sz,
                         const uint64_t* __restrict__ base, const uint64_t* __restrict__ deg,
                         const uint32_t* __restrict__ off, uint32_t fanout, uint64_t seed,
                         uint32_t hop, const int32_t* indices, int64_t* __restrict__ cand) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= sz[SZ_TOTAL]) return;
  const uint64_t nf = sz[SZ_NF];
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
// position of node c in this round, tagged with the round's epoch (a device counter) in the high
// word — a newer round's tag is always smaller, so the table is never cleared and graph replays
// stay correct.
__device__ __forceinline__ uint64_t round_tag(const uint64_t* sz) {
  return (uint64_t)(0xFFFFFFFFu - (uint32_t)sz[SZ_EPOCH]) << 32;
}

__global__ void k_next_round(uint64_t* epoch_dev, uint64_t* sz) {
  sz[SZ_EPOCH] = ++*epoch_dev;
}

__global__ void k_first(const int64_t* __restrict__ cand, const uint64_t* sz, uint64_t n_nodes,
                        const uint8_t* __restrict__ in_front, unsigned long long* firstpos,
                        unsigned long long* err) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= sz[SZ_TOTAL]) return;
  const uint64_t c = (uint64_t)cand[j];
  if (c >= n_nodes) {
    atomicMin(err, (unsigned long long)j);
    return;
  }
  if (!in_front[c]) atomicMin(firstpos + c, (unsigned long long)(round_tag(sz) | j));
}

__global__ void k_keep(const int64_t* __restrict__ cand, const uint64_t* sz, uint64_t n_nodes,
                       const uint8_t* __restrict__ in_front, const unsigned long long* __restrict__ firstpos,
                       uint32_t* __restrict__ keep) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= sz[SZ_TOTAL]) return;
  const uint64_t c = (uint64_t)cand[j];
  keep[j] = (c < n_nodes && !in_front[c] && firstpos[c] == (round_tag(sz) | j)) ? 1u : 0u;
}

__global__ void k_append(const int64_t* __restrict__ cand, const uint64_t* sz,
                         const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos,
                         int64_t* __restrict__ front, uint8_t* __restrict__ in_front) {
  const uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= sz[SZ_TOTAL] || !keep[j]) return;
  const int64_t c = cand[j];
  front[sz[SZ_NF] + pos[j]] = c;
  in_front[c] = 1;
}

__global__ void k_grow(uint64_t* sz) { sz[SZ_NF] += sz[SZ_ADDED]; }

__global__ void k_set(uint64_t* sz, int slot, uint64_t v) { sz[slot] = v; }

__global__ void k_finish(const uint64_t* sz, uint64_t* n_out) { *n_out = sz[SZ_NF]; }

__global__ void k_clear(const int64_t* __restrict__ front, const uint64_t* sz, uint8_t* __restrict__ in_front) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < sz[SZ_NF]) in_front[front[i]] = 0;
}

inline int blocks_for(uint64_t n, int per = 256) { return (int)std::max<uint64_t>(1, (n + per - 1) / per); }

}  // namespace

struct ut_graph {
  const int64_t* indptr = nullptr;
  const int32_t* indices = nullptr;
  uint64_t n_nodes = 0, n_edges = 0;
  Pin ip_pin, ix_pin;
  int indptr_hbm = 0;                    // ut_graph_set_option("indptr=hbm")
  int indices_hbm = 0;                   // ut_graph_set_option("indices=hbm")
  uint64_t launches = 0;                 // kernels enqueued by ut_sample*
  std::mutex mu;
  struct Dev {
    bool init = false;
    uint64_t indptr_dev = 0, indices_dev = 0;
    int64_t* indptr_copy = nullptr;      // HBM copy when indptr_hbm
    int32_t* indices_copy = nullptr;     // HBM copy when indices_hbm
    uint8_t* in_front = nullptr;         // n_nodes flags, all zero between calls
    unsigned long long* firstpos = nullptr;   // n_nodes epoch-tagged positions
    unsigned long long* err = nullptr;
    uint64_t* total_host = nullptr;      // pinned mirror for the synchronous API
    uint64_t* epoch_dev = nullptr;       // dedup round counter (device, graph-replay safe)
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
        (e = cudaMalloc(&s->epoch_dev, sizeof(uint64_t))) != cudaSuccess ||
        (e = cudaMallocHost(&s->total_host, 2 * sizeof(uint64_t))) != cudaSuccess) {
      cudaGetLastError();
      return set_err(UT_ENOMEM, "sampler state for %llu nodes", (unsigned long long)n);
    }
    cudaMemset(s->in_front, 0, n);
    cudaMemset(s->firstpos, 0xff, n * sizeof(unsigned long long));
    cudaMemset(s->err, 0xff, sizeof(unsigned long long));
    cudaMemset(s->epoch_dev, 0, sizeof(uint64_t));
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
    if ((e = cudaMemcpy(s->indptr_copy, g->indptr, bytes, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaStreamSynchronize(cudaStreamLegacy)) != cudaSuccess)   // landed before use
      return cuda_err(e, "indptr H2D");
  }
  if (g->indices_hbm && !s->indices_copy) {
    const uint64_t bytes = std::max<uint64_t>(1, g->n_edges) * sizeof(int32_t);
    if ((e = cudaMalloc(&s->indices_copy, bytes)) != cudaSuccess) {
      cudaGetLastError();
      return set_err(UT_ENOMEM, "HBM copy of indices (%llu bytes)", (unsigned long long)bytes);
    }
    if ((e = cudaMemcpy(s->indices_copy, g->indices, bytes, cudaMemcpyHostToDevice)) != cudaSuccess ||
        (e = cudaStreamSynchronize(cudaStreamLegacy)) != cudaSuccess)   // landed before use
      return cuda_err(e, "indices H2D");
  }
  *out = s;
  return UT_OK;
}

// Worst-case frontier sizes: every hop adds at most fanout new nodes per frontier node.
uint64_t frontier_cap(uint64_t n_seeds, const int32_t* fanouts, int hops, uint64_t n_nodes, int upto) {
  uint64_t c = n_seeds;
  for (int h = 0; h < upto && h < hops; ++h) c = std::min<uint64_t>(n_nodes, c + c * (uint64_t)fanouts[h]);
  return std::max<uint64_t>(c, 1);
}

template <typename T>
int pool_alloc(ut_graph::Dev* s, T** p, uint64_t count, cudaStream_t st) {
  *p = nullptr;
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
    if (!s.init && !s.indptr_copy && !s.indices_copy) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    cudaFree(s.in_front);
    cudaFree(s.firstpos);
    cudaFree(s.err);
    cudaFree(s.epoch_dev);
    cudaFreeHost(s.total_host);
    cudaFree(s.indptr_copy);
    cudaFree(s.indices_copy);
    if (s.pool) cudaMemPoolDestroy(s.pool);
  }
  cudaSetDevice(cur);
  unpin_host(&g->ip_pin);
  unpin_host(&g->ix_pin);
  delete g;
  return UT_OK;
}

uint64_t ut_graph_launches(const ut_graph* g) { return g ? g->launches : 0; }

int ut_graph_set_option(ut_graph* g, const char* opt) {
  if (!g || !opt) return set_err(UT_EINVAL, "NULL argument");
  if (!strcmp(opt, "indptr=hbm")) g->indptr_hbm = 1;
  else if (!strcmp(opt, "indptr=host")) g->indptr_hbm = 0;
  else if (!strcmp(opt, "indices=hbm")) g->indices_hbm = 1;
  else if (!strcmp(opt, "indices=host")) g->indices_hbm = 0;
  else return set_err(UT_EINVAL, "unknown option '%s'", opt);
  return UT_OK;
}

}  // extern "C"

namespace {

// Enqueue the whole sampler on `st`: no host synchronisation, launches sized by the worst case.
// `front` (capacity >= frontier_cap(all hops)) receives the node list, *n_dev its length.
int sample_enqueue(ut_graph* g, ut_graph::Dev* s, const int64_t* seeds_dev, uint64_t n_seeds,
                   const int32_t* fanouts, int n_hops, uint64_t seed, int64_t* front,
                   uint64_t* n_dev, cudaStream_t st) {
  const int64_t* indptr = g->indptr_hbm ? s->indptr_copy : (const int64_t*)s->indptr_dev;
  const int32_t* indices = g->indices_hbm ? s->indices_copy : (const int32_t*)s->indices_dev;
  uint64_t max_m = n_seeds;
  for (int h = 0; h < n_hops; ++h)
    max_m = std::max<uint64_t>(max_m, frontier_cap(n_seeds, fanouts, n_hops, g->n_nodes, h) * (uint64_t)fanouts[h]);
  const uint64_t fcap = frontier_cap(n_seeds, fanouts, n_hops, g->n_nodes, n_hops);
  if (max_m >= (1ull << 32) || fcap >= (1ull << 32)) return set_err(UT_EINVAL, "sampling bound exceeds 2^32");
  uint64_t* sz = nullptr;
  uint64_t *base = nullptr, *deg = nullptr;
  uint32_t *cnt = nullptr, *off = nullptr, *keep = nullptr, *pos = nullptr, *sums = nullptr;
  int64_t* cand = nullptr;
  int rc;
  if ((rc = pool_alloc(s, &sz, SZ_N, st)) != UT_OK || (rc = pool_alloc(s, &base, fcap, st)) != UT_OK ||
      (rc = pool_alloc(s, &deg, fcap, st)) != UT_OK || (rc = pool_alloc(s, &cnt, fcap, st)) != UT_OK ||
      (rc = pool_alloc(s, &off, fcap, st)) != UT_OK || (rc = pool_alloc(s, &keep, max_m, st)) != UT_OK ||
      (rc = pool_alloc(s, &pos, max_m, st)) != UT_OK ||
      (rc = pool_alloc(s, &sums, std::max(max_m, fcap) / kScanTile + 2, st)) != UT_OK ||
      (rc = pool_alloc(s, &cand, max_m, st)) != UT_OK)
    return rc;
  k_set<<<1, 1, 0, st>>>(sz, SZ_NF, 0);
  // merge `m_cap`-bounded candidates (count in sz[SZ_TOTAL]) into the frontier
  auto merge = [&](const int64_t* c, uint64_t m_cap) {
    k_next_round<<<1, 1, 0, st>>>(s->epoch_dev, sz);
    k_first<<<blocks_for(m_cap), 256, 0, st>>>(c, sz, g->n_nodes, s->in_front, s->firstpos, s->err);
    k_keep<<<blocks_for(m_cap), 256, 0, st>>>(c, sz, g->n_nodes, s->in_front, s->firstpos, keep);
    scan_u32(keep, pos, sz + SZ_TOTAL, m_cap, sz + SZ_ADDED, sums, st);
    k_append<<<blocks_for(m_cap), 256, 0, st>>>(c, sz, keep, pos, front, s->in_front);
    k_grow<<<1, 1, 0, st>>>(sz);
  };
  k_set<<<1, 1, 0, st>>>(sz, SZ_TOTAL, n_seeds);
  merge(seeds_dev, n_seeds);
  for (int h = 0; h < n_hops; ++h) {
    const uint32_t f = (uint32_t)fanouts[h];
    if (f == 0) continue;
    const uint64_t nf_cap = frontier_cap(n_seeds, fanouts, n_hops, g->n_nodes, h);
    const uint64_t m_cap = nf_cap * f;
    k_count<<<blocks_for(nf_cap), 256, 0, st>>>(front, sz, indptr, f, base, deg, cnt);
    scan_u32(cnt, off, sz + SZ_NF, nf_cap, sz + SZ_TOTAL, sums, st);
    k_sample<<<blocks_for(m_cap), 256, 0, st>>>(front, sz, base, deg, off, f, seed, (uint32_t)h,
                                                indices, cand);
    merge(cand, m_cap);
  }
  k_finish<<<1, 1, 0, st>>>(sz, n_dev);
  k_clear<<<blocks_for(fcap), 256, 0, st>>>(front, sz, s->in_front);
  // kernels: 2 k_set + merge (k_next_round, k_first, k_keep, 2-3 scan, k_append, k_grow) per
  // merge + (k_count, 2-3 scan, k_sample) per hop + k_finish + k_clear
  auto scan_k = [](uint64_t m) { return m > (uint64_t)kScanTile ? 3u : 2u; };
  uint64_t k = 2 + 2 + (5 + scan_k(n_seeds));
  for (int h = 0; h < n_hops; ++h) {
    if (!fanouts[h]) continue;
    const uint64_t nf_cap = frontier_cap(n_seeds, fanouts, n_hops, g->n_nodes, h);
    k += 2 + scan_k(nf_cap) + 5 + scan_k(nf_cap * (uint64_t)fanouts[h]);
  }
  g->launches += k;
  for (void* p : {(void*)sz, (void*)base, (void*)deg, (void*)cnt, (void*)off, (void*)keep,
                  (void*)pos, (void*)sums, (void*)cand})
    cudaFreeAsync(p, st);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return cuda_err(e, "sampler launch");
  return UT_OK;
}

int check_sample_args(ut_graph* g, const int64_t* seeds_dev, uint64_t n_seeds, const int32_t* fanouts,
                      int n_hops) {
  if (!g || (n_seeds && !seeds_dev) || (n_hops > 0 && !fanouts) || n_hops < 0)
    return set_err(UT_EINVAL, "NULL or negative argument");
  for (int h = 0; h < n_hops; ++h)
    if (fanouts[h] < 0) return set_err(UT_EINVAL, "fanout %d is negative", h);
  return UT_OK;
}

}  // namespace

extern "C" {

uint64_t ut_sample_capacity(uint64_t n_seeds, const int32_t* fanouts, int n_hops, uint64_t n_nodes) {
  if (n_seeds == 0 || (n_hops > 0 && !fanouts)) return n_seeds;
  return frontier_cap(n_seeds, fanouts, n_hops, n_nodes ? n_nodes : UINT64_MAX, n_hops);
}

int ut_sample_async(ut_graph* g, const int64_t* seeds_dev, uint64_t n_seeds, const int32_t* fanouts,
                    int n_hops, uint64_t seed, int64_t* nodes_dev, uint64_t cap, uint64_t* n_out_dev,
                    ut_stream_t stream) {
  int rc = check_sample_args(g, seeds_dev, n_seeds, fanouts, n_hops);
  if (rc != UT_OK) return rc;
  if (!n_out_dev || !nodes_dev) return set_err(UT_EINVAL, "NULL nodes_dev / n_out_dev");
  const uint64_t need = ut_sample_capacity(n_seeds, fanouts, n_hops, g->n_nodes);
  if (cap < need) return set_err(UT_EINVAL, "nodes capacity %llu < worst case %llu",
                                 (unsigned long long)cap, (unsigned long long)need);
  cudaStream_t st = (cudaStream_t)stream;
  if (n_seeds == 0) {
    k_set<<<1, 1, 0, st>>>(n_out_dev, 0, 0);
    return UT_OK;
  }
  std::lock_guard<std::mutex> lk(g->mu);
  ut_graph::Dev* s;
  if ((rc = graph_dev(g, &s)) != UT_OK) return rc;
  return sample_enqueue(g, s, seeds_dev, n_seeds, fanouts, n_hops, seed, nodes_dev, n_out_dev, st);
}

int ut_sample(ut_graph* g, const int64_t* seeds_dev, uint64_t n_seeds, const int32_t* fanouts,
              int n_hops, uint64_t seed, int64_t* nodes_dev, uint64_t cap, uint64_t* n_out,
              ut_stream_t stream) {
  int rc = check_sample_args(g, seeds_dev, n_seeds, fanouts, n_hops);
  if (rc != UT_OK) return rc;
  if (!n_out) return set_err(UT_EINVAL, "NULL n_out");
  *n_out = 0;
  if (n_seeds == 0) return UT_OK;
  std::lock_guard<std::mutex> lk(g->mu);
  ut_graph::Dev* s;
  if ((rc = graph_dev(g, &s)) != UT_OK) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const uint64_t fcap = ut_sample_capacity(n_seeds, fanouts, n_hops, g->n_nodes);
  int64_t* front = nodes_dev;
  const bool own = cap < fcap || !nodes_dev;
  uint64_t* n_dev = nullptr;
  if ((rc = pool_alloc(s, &n_dev, 1, st)) != UT_OK) return rc;
  if (own && (rc = pool_alloc(s, &front, fcap, st)) != UT_OK) return rc;
  rc = sample_enqueue(g, s, seeds_dev, n_seeds, fanouts, n_hops, seed, front, n_dev, st);
  cudaError_t e = cudaSuccess;
  if (rc == UT_OK) {
    cudaMemcpyAsync(&s->total_host[0], n_dev, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&s->total_host[1], s->err, sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) rc = cuda_err(e, "sampler");
  }
  if (rc == UT_OK) {
    const uint64_t n = s->total_host[0];
    *n_out = n;
    if (s->total_host[1] != ~0ull) {
      cudaMemsetAsync(s->err, 0xff, sizeof(unsigned long long), st);
      rc = set_err(UT_ERANGE, "seed %llu is out of range", (unsigned long long)s->total_host[1]);
    } else if (own) {
      if (n > cap || !nodes_dev)
        rc = set_err(UT_EINVAL, "nodes buffer holds %llu, need %llu", (unsigned long long)cap,
                     (unsigned long long)n);
      else if ((e = cudaMemcpyAsync(nodes_dev, front, n * sizeof(int64_t), cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        rc = cuda_err(e, "copy nodes");
    }
  }
  if (own) cudaFreeAsync(front, st);
  cudaFreeAsync(n_dev, st);
  return rc;
}

}  // extern "C"
