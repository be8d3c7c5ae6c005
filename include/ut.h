/*
 * ut.h — C ABI of the B200 unified-tensor gather (PyTorch-Direct, arXiv 2101.07956).
 *
 * The operation. PyTorch-Direct keeps the node-feature table in host memory as a "unified
 * tensor" that GPU threads dereference directly over the host link (PAPER.md:239-243,
 * §3 Fig. 2b; §4.1), and its hot path is "indexing unified tensor with GPU
 * tensor", `unified_tensor[gpu_tensor]` (Table 1; Listing 2),
 * whose output is a GPU tensor (Table 3 row 2 / col 1). The feature table is
 * "a 2D array where the row indices are the IDs of nodes and the columns are the features of
 * each node". This library computes exactly
 *
 *     for i in [0, n):  out[i*rb .. (i+1)*rb) = table[idx[i]*rb .. (idx[i]+1)*rb)
 *
 * byte for byte (rb = row_bytes), with GPU threads reading the rows straight out of the
 * host-pinned, device-mapped table: no CPU gather and no staging DMA (contrast PAPER.md:221-225,
 * Fig. 2a). The paper's alignment optimisation (§4.5) changes the access
 * order, never the result ("the output indices are also identically adjusted to maintain the
 * ordering"); here every kernel variant must be bit-identical to the loop above.
 *
 * Layout. The table is rows x rb bytes, row-major, dense, starting at host_ptr (any alignment).
 * idx is int64 (reading R2; the 4-B sweep table has 2^32 rows). out is n x rb bytes,
 * row-major, dense, in device memory (any alignment; 16-B aligned is the fast path).
 *
 * Errors. Functions return UT_OK (0) or a negative ut_status; ut_register returns NULL on
 * failure. The reason of the last failure on the calling thread is in ut_last_error().
 * An out-of-range or negative idx[i] is NOT a synchronous error (the kernel is asynchronous):
 * that output row is zero-filled and the smallest such position i is recorded in a
 * per-table, per-device error word that ut_error_pos() reads and clears (DESIGN.md reading
 * R4, following SPEC.md:151 "index error naming the offending position").
 *
 * Threading. Concurrent ut_gather calls on one table from any thread, stream or device are
 * safe (the table is read-only). ut_release must not race with in-flight gathers.
 */
#ifndef UT_H
#define UT_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define UT_API __attribute__((visibility("default")))
#else
#define UT_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Opaque, process-local handle of one registered table. */
typedef struct ut_table ut_table;

/* Same type as cudaStream_t (`struct CUstream_st*`); NULL = the legacy default stream. */
typedef struct CUstream_st* ut_stream_t;

typedef enum ut_status {
  UT_OK = 0,
  UT_EINVAL = -1,   /* bad argument: NULL pointer, zero size, overflow, unknown plan name     */
  UT_ENOMEM = -2,   /* host registration or device scratch allocation failed                */
  UT_ECUDA = -3,    /* a CUDA runtime call or kernel launch failed (message has the reason)  */
  UT_ERANGE = -4,   /* ut_error_pos only: an out-of-range index was recorded                 */
  UT_ENOTSUP = -5   /* the device cannot map host memory                                     */
} ut_status;

/*
 * ut_register — make `rows * row_bytes` bytes at host_ptr GPU-addressable in place.
 * The paper's `features = dataload().to("unified")` (Listing 2 line 2; Table 1
 * PAPER.md:373) copies into a new unified allocation (§4.4); this entry
 * instead pins and maps the caller's memory WITHOUT copying, so that several processes can
 * register one shared table (reading R1).
 *   host_ptr   caller-owned host memory, any alignment. It must stay valid, and unmodified while
 *              any gather is in flight, until ut_release. If it lies inside one page-locked and
 *              mapped allocation (cudaHostAlloc / cudaHostRegister by the caller), it is adopted
 *              and left pinned on release; otherwise its pages are registered with
 *              cudaHostRegister(Portable|Mapped[|ReadOnly when the device supports it]) and
 *              unregistered by ut_release. A range that only partly overlaps pinned memory (other
 *              allocations' pages at its ends or inside it) is walked allocation by allocation:
 *              the pinned stretches are adopted and every unpinned gap is registered, so every
 *              byte is GPU-addressable before the handle is returned (or the call fails).
 *   rows       number of rows, >= 1.
 *   row_bytes  bytes per row, >= 1; rows * row_bytes must not overflow 64 bits.
 * The current CUDA device is used for registration; the mapping is Portable, so the handle
 * serves every device of the process. Registration pins whole pages: the table should not share
 * its first or last page with host buffers that other code hands to CUDA copies (allocate big
 * tables page-aligned, e.g. mmap); pages already pinned by a neighbour are left to it. Returns NULL on failure (UT_EINVAL / UT_ENOMEM /
 * UT_ECUDA / UT_ENOTSUP via ut_last_error).
 */
UT_API ut_table* ut_register(const void* host_ptr, uint64_t rows, uint64_t row_bytes);

/*
 * ut_create — the paper's own form, `t.to("unified")` (Table 1; §4.4
 * P:530-531 "a new memory allocator ... for all unified tensors"): allocate a NEW host-resident
 * table that the GPU maps, copy `src` into it (src may be NULL: the caller fills *host_out), and
 * return its handle. Kinds (SURVEY NEXT-4 registration variants):
 *   UT_ALLOC_PINNED    cudaHostAlloc(Portable|Mapped) page-locked host memory;
 *   UT_ALLOC_MANAGED   cudaMallocManaged + cudaMemAdvise(SetPreferredLocation = CPU,
 *                      SetAccessedBy = current device): the paper's default advice for unified
 *                      tensors (Table 2) — data stays in host memory, GPU maps it;
 *   UT_ALLOC_VMM_HOST  cuMemCreate(location HOST_NUMA of the current device) in 2-MiB granules,
 *                      mapped read/write for the device and the host.
 * *host_out receives the host (= device, UVA) address of the rows * row_bytes bytes; the memory
 * is owned by the table and freed by ut_release. The handle serves every device of the process
 * (one table per box, one host thread per GPU): the first call on another device extends the
 * mapping to it — SetAccessedBy(that device) for MANAGED, cuMemSetAccess for VMM_HOST (UT_ENOTSUP
 * if the driver refuses); PINNED memory is Portable already. Returns NULL on failure (UT_EINVAL /
 * UT_ENOMEM / UT_ECUDA / UT_ENOTSUP via ut_last_error).
 */
typedef enum ut_alloc_kind {
  UT_ALLOC_PINNED = 0,
  UT_ALLOC_MANAGED = 1,
  UT_ALLOC_VMM_HOST = 2,
  UT_ALLOC_SYSTEM = 3     /* ut_pool only: plain malloc, NOT GPU-mapped — exercises the pool's
                             bookkeeping without a GPU; ut_create / ut_pool_table refuse it    */
} ut_alloc_kind;

UT_API ut_table* ut_create(const void* src, uint64_t rows, uint64_t row_bytes, int kind,
                           void** host_out);

/*
 * The unified allocator with block recycling (reading
 * R19). PAPER.md §4.4: "A new memory allocator is implemented to govern the memory
 * allocation for all unified tensors. It adapts the allocation recycling mechanism from the
 * PyTorch CUDA allocator to reduce the number of CUDA API invocations."
 *
 * ut_pool_create — a pool of host blocks of one kind: UT_ALLOC_PINNED or UT_ALLOC_MANAGED (the
 *   same backend calls and advice as ut_create, on the device current at this call), or
 *   UT_ALLOC_SYSTEM (malloc; bookkeeping only, usable without a GPU). limit_bytes bounds the
 *   bytes the pool holds from its backend, live + cached (0 = no limit). NULL on failure
 *   (UT_EINVAL unknown kind / UT_ENOMEM / UT_ECUDA via ut_last_error).
 * ut_pool_alloc — *host_out = a block of *capacity_out = bytes rounded up to a multiple of 512
 *   (capacity_out may be NULL). The most recently freed cached block of exactly that capacity is
 *   reused with no CUDA call; otherwise the backend allocates one. A backend allocation that would
 *   pass limit_bytes (or that the backend refuses) first returns every cached block to the backend
 *   and is retried once. bytes == 0 gives *host_out = NULL, capacity 0, no backend call. Blocks
 *   are not zeroed. Returns UT_OK, UT_EINVAL (NULL pool / host_out), UT_ENOMEM or UT_ECUDA.
 * ut_pool_free — cache a live block (never returned to the backend here); NULL is a no-op.
 *   UT_EINVAL if host is not a live block of this pool (double free, foreign pointer). The caller
 *   guarantees no GPU work still reads or writes the block (the pool does not synchronise).
 * ut_pool_release_cached — return every cached block to the backend (cudaFreeHost / cudaFree).
 * ut_pool_get_stats — counters, see ut_pool_stats.
 * ut_pool_destroy — release the cached blocks and the pool. UT_EINVAL (pool unchanged) while
 *   any block is live, including the blocks of live pool tables. NULL is a no-op.
 * The pool is thread-safe (one mutex; backend calls happen under it).
 */
typedef struct ut_pool ut_pool;

typedef struct ut_pool_stats {
  uint64_t backend_calls;    /* fresh backend allocations (cudaHostAlloc / cudaMallocManaged)   */
  uint64_t backend_frees;    /* blocks returned to the backend (release_cached, limit, destroy) */
  uint64_t recycled_hits;    /* requests served from the cache                                 */
  uint64_t bytes_live;       /* capacity of the blocks in use                                   */
  uint64_t bytes_cached;     /* capacity of the cached blocks                                   */
  uint64_t blocks_live;
  uint64_t blocks_cached;
  uint64_t limit_bytes;      /* as created; 0 = none                                            */
} ut_pool_stats;

UT_API ut_pool* ut_pool_create(int kind, uint64_t limit_bytes);
UT_API int ut_pool_alloc(ut_pool* p, uint64_t bytes, void** host_out, uint64_t* capacity_out);
UT_API int ut_pool_free(ut_pool* p, void* host);
UT_API int ut_pool_release_cached(ut_pool* p);
UT_API int ut_pool_get_stats(const ut_pool* p, ut_pool_stats* stats);
UT_API int ut_pool_destroy(ut_pool* p);

/*
 * ut_pool_table — ut_create's table (`t.to("unified")`) over a block of pool p (kind PINNED or
 * MANAGED): rows * row_bytes bytes taken with ut_pool_alloc, src copied in when not NULL,
 * *host_out = the block. ut_release on the table hands the block back to p (cached, no CUDA free
 * call); p must outlive the table. Mapping on other devices as for ut_create. Returns NULL on
 * failure (UT_EINVAL: NULL p / host_out, zero rows or row_bytes, overflow, SYSTEM kind;
 * UT_ENOMEM / UT_ECUDA / UT_ENOTSUP via ut_last_error).
 */
UT_API ut_table* ut_pool_table(ut_pool* p, const void* src, uint64_t rows, uint64_t row_bytes,
                               void** host_out);

/*
 * ut_gather — out_dev[i*rb .. (i+1)*rb) = row idx_dev[i] of the table, for i in [0, n).
 * The paper's `input_features = features[neighbor_id]` with a GPU index
 * tensor and a GPU output.
 *   t        handle from ut_register.
 *   idx_dev  n int64 row ids in device memory of the CURRENT device (caller-owned, read-only).
 *   n        number of rows to gather; n == 0 returns UT_OK without launching anything and
 *            leaves out_dev untouched.
 *   out_dev  >= n*rb bytes of device memory on the current device, not overlapping idx_dev
 *            (caller-owned). Any alignment.
 *   stream   stream to enqueue on; the call is asynchronous and stream-ordered, so a consumer
 *            kernel on the same stream sees the rows.
 * Reads touch only table bytes in [host_ptr, host_ptr + rows*rb) (reading R8).
 * Returns UT_OK, UT_EINVAL (NULL t/idx/out with n > 0, n*rb overflow) or UT_ECUDA.
 */
UT_API int ut_gather(const ut_table* t, const int64_t* idx_dev, uint64_t n, void* out_dev,
              ut_stream_t stream);

/*
 * ut_gather_i32 — ut_gather with 32-bit row ids (a GPU index tensor of dtype int32, which
 * PyTorch's indexing also accepts; reading R2 keeps int64 as the native form because
 * the 4-B sweep table has 2^32 rows). The ids are sign-extended into stream-ordered library
 * scratch (12 B of HBM traffic per row, one small launch) and gathered exactly as ut_gather
 * does: the same bytes, the same out-of-range rule (a negative id is out of range; its row is
 * zero-filled and its position recorded for ut_error_pos). Arguments, layout, ownership and
 * errors as ut_gather, plus UT_ENOMEM when the scratch cannot be allocated.
 */
UT_API int ut_gather_i32(const ut_table* t, const int32_t* idx_dev, uint64_t n, void* out_dev,
                         ut_stream_t stream);

/*
 * ut_gather_dn — ut_gather whose row count lives in device memory: gathers
 * min(*n_dev, max_n) rows, read by the kernels themselves, so a device-side producer of the index
 * list (ut_sample_async) and this gather need no host synchronisation between them and can be
 * captured in one CUDA graph. Launch sizes follow max_n (< 2^31). Errors as ut_gather.
 */
UT_API int ut_gather_dn(const ut_table* t, const int64_t* idx_dev, const uint64_t* n_dev,
                        uint64_t max_n, void* out_dev, ut_stream_t stream);

/*
 * ut_gather_multi — the box form: one host thread enqueues one gather on each of `count` devices
 * over the ONE table (every GPU of the box pulling its own minibatch over its own link,
 * PAPER.md:239-243). For k in [0, count): device devs[k] runs
 * ut_gather(t, idx_dev[k], n[k], out_dev[k], streams[k]) — idx_dev[k] / out_dev[k] in that
 * device's memory, streams[k] a stream of that device (NULL: its legacy default stream).
 * Asynchronous like ut_gather; the calling thread's current device is restored. The first
 * failing entry stops the call: its error is returned and the entries before it stay enqueued.
 * A library-owned table (ut_create) is mapped for each device on first use (see ut_create);
 * a registered table is Portable. Returns UT_OK, UT_EINVAL (count < 1, NULL arrays) or the
 * failing entry's ut_gather error.
 */
UT_API int ut_gather_multi(const ut_table* t, int count, const int* devs,
                           const int64_t* const* idx_dev, const uint64_t* n,
                           void* const* out_dev, const ut_stream_t* streams);

/*
 * ut_gather_host — the same gather from and to HOST buffers (the end-to-end form).
 *   idx_host  n int64 row ids in host memory (page-locked for full speed; caller-owned).
 *   out_host  >= n*rb bytes of host memory (caller-owned).
 * If out_host is page-locked and mapped (cudaHostAlloc / cudaHostRegister'ed), idx is copied to
 * the device and the gather kernel stores the rows straight into out_host over the link (one
 * pass, no HBM round trip); every byte of [out_host, out_host + n*rb) must then be mapped (one
 * allocation, or adjacent ones under UVA — checked allocation by allocation before any work), and
 * a buffer whose first byte is page-locked but whose range is not returns UT_EINVAL (kernel
 * stores would fault in the unlocked stretch, and the copy engine refuses a partly locked
 * destination). Otherwise (pageable memory) rows are gathered in
 * chunks into library-owned device
 * scratch and copied back by the copy engine on a second stream, overlapping the two link
 * directions (UT_HOST_PIPELINE=1 forces this path). Device scratch is owned by the table and
 * grown on demand (x1.5 in whole MiB, since a reallocation synchronises the device).
 * Synchronous: returns after out_host holds the result, on `stream`. Calls on different devices
 * run concurrently; calls on the same device serialise (they share that device's scratch).
 * Out-of-range handling as ut_gather. Returns UT_OK, UT_EINVAL, UT_ENOMEM or UT_ECUDA.
 */
UT_API int ut_gather_host(const ut_table* t, const int64_t* idx_host, uint64_t n, void* out_host,
                   ut_stream_t stream);

/*
 * ut_release — free the handle; unregister the memory iff ut_register registered it; free a
 * ut_create table's memory, or hand a ut_pool_table's block back to its pool (cached).
 * The table's device error words return to the per-device slab every table of the process
 * shares; the shared stream-ordered scratch pool is trimmed when the device's last table goes.
 * NULL is a no-op returning UT_OK.
 * Must not be called while a gather on the table is in flight.
 */
UT_API int ut_release(ut_table* t);

/*
 * ut_error_pos — synchronise `stream`, then report and clear the smallest position i whose
 * idx[i] was out of range (< 0 or >= rows) in any gather on the current device since the last
 * call. *first_bad = -1 and UT_OK if none; *first_bad = i and UT_ERANGE otherwise.
 */
UT_API int ut_error_pos(const ut_table* t, ut_stream_t stream, int64_t* first_bad);

/*
 * ut_last_error — copy the calling thread's last error message (NUL-terminated, truncated to
 * cap) into msg (may be NULL when cap == 0) and return its ut_status code.
 */
UT_API int ut_last_error(char* msg, size_t cap);

/*
 * ut_plan_name — name of the kernel variant ut_gather uses on this table for a 16-B aligned
 * out_dev, e.g. "vec16.g32", "realign.g32x", "narrow4". The string is
 * static. Returns "invalid" for NULL.
 */
UT_API const char* ut_plan_name(const ut_table* t);

/*
 * ut_plan_probe — the variant ut_gather would pick for a table at host address `base` with
 * `rows` x `row_bytes` and an output at device address `out` (no CUDA call; for tests and
 * reports). Returns the static plan name, or "invalid" for zero sizes.
 */
UT_API const char* ut_plan_probe(uint64_t base, uint64_t rows, uint64_t row_bytes, uint64_t out);

/*
 * ut_set_plan — force a kernel variant by kind for A/B measurement: "narrow", "vec16",
 * "vec16x", "realign", "realignx", the TMA variants "bulk" (1-D bulk copy per row) and "tma4"
 * (tensor-map tile::gather4, 4 rows per instruction), the paper's "paper_naive" / "paper_shift",
 * or "auto" (the default choice). A kind whose preconditions
 * the table violates returns UT_EINVAL and leaves the plan unchanged; every admissible kind is
 * correct for any output alignment (ut_gather falls back to "auto" for an output it cannot take).
 * "timing=on|off" brackets each gather-kernel launch with CUDA events (see ut_get_stats).
 * "runs=on|off" (default off): for 16-B aligned tables, sort the rows exactly and copy runs of
 * table-adjacent rows with one warp so shared boundary lines are requested once.
 * "share=on|off|auto": neighbour line sharing for 16-B aligned tables with 128 < rb <= 512 —
 * the warp of a selected row also fetches its selected successor's bytes in the 128-B line the
 * two share, so the line is requested once; auto = on for gathers of >= 64K rows
 * that select >= 1/16 of the table (host-known row counts only). Costs a hash of the selection,
 * 8 B x 2^ceil(log2 2n), of stream-ordered scratch per gather (O(n), independent of the table).
 * "exact=on|off|auto" (auto = off): with the reorder, sort the work items of each 2-MiB bucket
 * exactly by row id (an A/B knob: measured no gain).
 * "stage=on|off|auto" (auto = off): ut_gather_host's direct path gathers tiles of consecutive
 * output rows into shared memory and writes each tile's span with whole-line stores (k_staged;
 * an A/B knob — measured no gain).
 * "conc=auto|dense|sparse" picks the launch shape: dense = every SM full of warps; sparse = a
 * quarter of the SMs, one row-step per warp (fewer translation pages in flight); auto = sparse
 * for reordered gathers from tables > 1 GiB.
 * "reorder=on|off|auto" controls the translation-locality stage instead:
 * work items are visited grouped by the 2-MiB table region their row lies in, the output order
 * is unchanged; "auto" enables it for gathers of >= 64K rows narrower than 4 KiB from tables
 * > 1 GiB (or > 64 MiB for rows <= 128 B; not for managed tables unless rows <= 128 B).
 * The environment variables UT_PLAN and UT_REORDER, read at ut_register, do the same.
 */
UT_API int ut_set_plan(ut_table* t, const char* name);

/*
 * ut_mem_advise — the paper's `unified_tensor.memAdvise(advise, adviseDevice)` (Table 2,
 * PAPER.md:413-416, 440-450): apply cudaMemAdvise to the table's storage and return the CUDA
 * error code as an int (0 = cudaSuccess) — "Invoke cudaMemAdvise and returns error code".
 *   advice  0 SetPreferredLocation, 1 UnsetPreferredLocation, 2 SetAccessedBy,
 *           3 UnsetAccessedBy, 4 SetReadMostly, 5 UnsetReadMostly.
 *   device  -1 = the CPU (host), >= 0 = that GPU.
 * Meaningful for managed tables (ut_create UT_ALLOC_MANAGED); pinned memory returns the runtime's
 * error code (cudaErrorInvalidValue) unchanged. Returns UT_EINVAL (negative) for a NULL table or
 * an unknown advice.
 */
UT_API int ut_mem_advise(const ut_table* t, int advice, int device);

/*
 * ut_numa_interleave — stripe a managed table's host pages round-robin over host NUMA nodes
 * 0..nodes-1 (the box's one shared table is "NUMA-interleaved by default", so on a
 * two-socket box each socket's GPUs read half their rows from local DRAM and neither socket's
 * memory carries the whole box's gather traffic). It is the paper's memAdvise interface (Table 2,
 * PAPER.md:413-416) with CUDA's host-NUMA location: stripe k of `chunk_bytes` gets
 * cudaMemAdvise(SetPreferredLocation, {HostNuma, k mod nodes}); SetAccessedBy is unchanged, so
 * GPUs keep reading the pages in place over the link. The advice places pages when they are first
 * populated: call it between ut_create(src = NULL) and the first write of the table.
 *   t            a UT_ALLOC_MANAGED table.
 *   nodes        >= 1 host NUMA nodes, ids 0..nodes-1 (nodes == 1: the whole table on node 0).
 *   chunk_bytes  stripe size, rounded up to a multiple of 2 MiB (the managed-memory block);
 *                0 = 2 MiB.
 * The placement is read back (cudaMemRangeGetAttribute) on the first stripe of every node.
 * Returns UT_OK, UT_EINVAL (NULL table, nodes < 1), UT_ENOTSUP (not a managed table, or the
 * driver accepted the advice without applying it — measured on this pool's virtualised boxes) or
 * UT_ECUDA (the runtime refused the advice, e.g. a node id the host does not have). On either
 * error the whole table is advised back to SetPreferredLocation = CPU, the state ut_create left
 * it in.
 */
UT_API int ut_numa_interleave(const ut_table* t, int nodes, uint64_t chunk_bytes);

/*
 * ut_numa_place — put a whole managed table on ONE host NUMA node ("one replica per
 * socket if RAM allows, so every GPU reads locally": the caller creates one table per node,
 * places replica k on node k with this call, fills it, and has each GPU gather from the replica
 * on its own node). cudaMemAdvise(SetPreferredLocation, {HostNuma, node}) over the table
 * (PAPER.md:413-416's memAdvise with CUDA's host-NUMA location); SetAccessedBy is unchanged.
 * Call it between ut_create(src = NULL) and the first write, like ut_numa_interleave.
 *   t     a UT_ALLOC_MANAGED table.
 *   node  host NUMA node id >= 0.
 * The placement is read back at the table's first page. Returns UT_OK, UT_EINVAL (NULL table,
 * node < 0), UT_ENOTSUP (not a managed table, or the driver accepted the advice without applying
 * it) or UT_ECUDA (the runtime refused the advice, e.g. a node the host does not have). On either
 * error the table is advised back to SetPreferredLocation = CPU; the caller may then place it by
 * first touch from that node's CPUs instead (bench.py --numa replica does).
 */
UT_API int ut_numa_place(const ut_table* t, int node);

/* ---- GPU-side neighbour sampling over a host-resident CSR graph -------------
 * The step before the gather that the paper leaves on the CPU. The CSR stays in
 * host memory (pinned in place like a feature table) and GPU threads read it over the link. */
typedef struct ut_graph ut_graph;

/*
 * ut_graph_register — pin a CSR graph in place for GPU sampling.
 *   indptr   int64[n_nodes + 1], indptr[0] == 0, non-decreasing, indptr[n_nodes] == n_edges.
 *   indices  int32[n_edges] neighbour ids in [0, n_nodes) (the caller guarantees the range).
 *   n_nodes  in [1, 2^31).
 * Both arrays are caller-owned and must stay valid and unmodified until ut_graph_release. The
 * current device gets n_nodes bytes + 8*n_nodes bytes of sampler state. NULL on failure.
 */
UT_API ut_graph* ut_graph_register(const int64_t* indptr, const int32_t* indices, uint64_t n_nodes,
                                   uint64_t n_edges);

/* "indptr=hbm" keeps a device copy of indptr (8*(n_nodes+1) bytes) so only `indices` is read
 * over the link; "indices=hbm" keeps a device copy of indices (4*n_edges bytes); "...=host"
 * (the default for both) reads that array over the link. */
UT_API int ut_graph_set_option(ut_graph* g, const char* option);

/*
 * ut_sample — multi-hop neighbour sampling, reading R17 (= oracle/ut_oracle_sample.c):
 * frontier_0 = seeds (first-appearance unique); at hop h each frontier node v takes
 * min(deg(v), fanouts[h]) distinct neighbour slots (all when deg <= fanout, else one per stratum
 * [floor(t*deg/f), floor((t+1)*deg/f)) chosen by the counter hash H(seed, h, v, t)); the next
 * frontier is the old one followed by the not-yet-seen sampled neighbours in (v, t) order.
 *   seeds_dev  n_seeds int64 node ids on the current device.
 *   fanouts    n_hops host ints >= 0.
 *   nodes_dev  device int64[cap]: receives the final frontier (the minibatch's node list, seeds
 *              first) — the index list a following ut_gather reads.
 *   *n_out     node count (set even when cap is too small, then UT_EINVAL is returned).
 * Synchronises `stream` once, at the end, to return the count (the sampler itself keeps every
 * size in device memory). Returns UT_OK, UT_EINVAL, UT_ERANGE (a seed outside [0, n_nodes); such
 * seeds are dropped), UT_ENOMEM or UT_ECUDA.
 * Concurrency: ONE sample in flight per graph per device. The sampler's device state (frontier
 * marks, dedup table, round counter) is per graph and device, so calls on one graph must be
 * ordered on the device — issue them on one stream, or make the next call's stream wait for the
 * previous one (this includes overlapping replays of a captured ut_sample_async). Different
 * graphs, or different devices, are independent. (Unlike ut_gather, which is read-only on its
 * table and safe from any number of streams.)
 */
UT_API int ut_sample(ut_graph* g, const int64_t* seeds_dev, uint64_t n_seeds, const int32_t* fanouts,
                     int n_hops, uint64_t seed, int64_t* nodes_dev, uint64_t cap, uint64_t* n_out,
                     ut_stream_t stream);

/*
 * ut_sample_capacity — the worst-case node count of a call: min(n_nodes, n_seeds * prod(1 + f_h)).
 * ut_sample_async needs nodes_dev to hold this many entries.
 */
UT_API uint64_t ut_sample_capacity(uint64_t n_seeds, const int32_t* fanouts, int n_hops,
                                   uint64_t n_nodes);

/*
 * ut_sample_async — ut_sample with no host synchronisation: every launch is sized by the
 * worst case and reads the live sizes from device memory; the node count is written to the
 * device word *n_out_dev. cap must be >= ut_sample_capacity(...). Seeds outside [0, n_nodes) are
 * dropped silently. With ut_gather_dn(t, nodes_dev, n_out_dev, cap, ...) on the same stream, a
 * whole minibatch (sample + gather) is host-sync-free and can be captured in a CUDA graph;
 * replays re-read the seeds buffer. Returns UT_OK, UT_EINVAL, UT_ENOMEM or UT_ECUDA.
 */
UT_API int ut_sample_async(ut_graph* g, const int64_t* seeds_dev, uint64_t n_seeds,
                           const int32_t* fanouts, int n_hops, uint64_t seed, int64_t* nodes_dev,
                           uint64_t cap, uint64_t* n_out_dev, ut_stream_t stream);

/* Kernels enqueued by ut_sample / ut_sample_async on this graph so far (for launch counts). */
UT_API uint64_t ut_graph_launches(const ut_graph* g);

/* Free the sampler state and unpin the CSR arrays (if ut_graph_register pinned them). */
UT_API int ut_graph_release(ut_graph* g);

/* Per-device counters of one table (for reports and the bench's launch count). */
typedef struct ut_stats {
  uint64_t gathers;          /* gather-kernel launches (one per ut_gather, per chunk of ut_gather_host) */
  uint64_t kernel_launches;  /* every kernel this library launched (gather + reorder stage)           */
  uint64_t rows;             /* rows gathered                                                        */
  uint64_t bytes;            /* rows * row_bytes                                                     */
  uint64_t timed_launches;   /* gather-kernel launches bracketed by events ("timing=on")            */
  double gather_kernel_ms;   /* their summed device time (CUDA events on the launch stream)          */
  uint64_t share_gathers;    /* gathers that took neighbour line sharing ("share")    */
} ut_stats;

/*
 * ut_get_stats — counters of table t on the current device since registration or the last
 * reset. With "timing=on" (ut_set_plan) every gather-kernel launch is bracketed by CUDA events
 * on its stream; this call waits for the pending events and adds their durations. reset != 0
 * zeroes the counters afterwards. Returns UT_OK, UT_EINVAL or UT_ECUDA.
 */
UT_API int ut_get_stats(const ut_table* t, ut_stats* stats, int reset);

/* Table facts recorded at registration (for tests and reports). */
typedef struct ut_table_info {
  uint64_t rows;
  uint64_t row_bytes;
  uint64_t host_addr;     /* host_ptr as an integer                                        */
  uint64_t dev_addr;      /* device address of host_ptr on the registering device          */
  int registered;         /* 1 if ut_register pinned the memory, 0 if it adopted it          */
  int alloc_kind;         /* ut_alloc_kind for ut_create tables, -1 for caller memory       */
  int read_only;          /* 1 if registered with cudaHostRegisterReadOnly                   */
  int base_mod128;        /* host_ptr mod 128                                               */
  int device;             /* device that was current at registration                        */
} ut_table_info;

/* Fill *info. Returns UT_OK or UT_EINVAL. */
UT_API int ut_table_get_info(const ut_table* t, ut_table_info* info);

/* ============================================================================================
 * Cooperative multi-rank gather.
 *
 * Several ranks (one process per GPU, or several processes sharing a GPU) gather their own
 * minibatches from one host table in the same step. The paper has each GPU read its rows over
 * its own link (Fig. 2b), so rows sampled by several ranks cross the host side
 * once per rank. Here the table's rows are split into blocks owned round-robin by the ranks
 * (ut_coop_owner); a step sends each index to its owner (P2P stores into the owner's inbox in
 * device memory), each owner fetches the union of the rows it was asked for ONCE from host memory
 * with ut_gather_dn, and each rank copies its rows from the owners' staging rows (P2P loads) into
 * its output in index order. The result is exactly ut_gather's: out[i*rb..(i+1)*rb) = row idx[i]
 * (PAPER.md:377); out-of-range indices give a zero row and a recorded position (reading R4).
 *
 * Setup: every rank calls ut_coop_create (same world, max_n and table shape on every rank; each
 * rank registers the table itself), ut_coop_export, moves the handles to every rank (the caller's
 * plumbing, e.g. torch.distributed all_gather_object), then ut_coop_open with all handles in rank
 * order. A step is either
 *   (a) ut_coop_gather on every rank: phases synchronised on the device (stream memory
 *       operations on flag words in peer memory; no host round trip), or
 *   (b) ut_coop_dispatch; [stream sync + host barrier of all ranks]; ut_coop_fetch;
 *       [stream sync + host barrier]; ut_coop_combine — the caller synchronises.
 * Every rank must take part in every step (n may be 0). Buffers are double-buffered by step
 * parity, so consecutive steps need no extra barrier. Not thread-safe per handle.
 * ============================================================================================ */
typedef struct ut_coop ut_coop;

#define UT_COOP_HANDLE_BYTES 64

/* Create this rank's side on the CURRENT device. t: this process's handle of the shared table.
 * world in [1, 64], rank in [0, world); max_n: the largest n any rank passes per step, with
 * world*max_n < 2^31. Allocates the rank's symmetric device region (2 x (inboxes world*max_n*12 B
 * + staging world*max_n*rb B)) and private scratch (a dedup tag table of ~rows/world x 8 B).
 * world == 1 needs no ut_coop_open. NULL on failure (ut_last_error). */
UT_API ut_coop* ut_coop_create(const ut_table* t, int world, int rank, uint64_t max_n);

/* Partitioned form: the host table is never held whole by any process. `part` holds only the
 * rows this rank owns, in its local order (row l = table row ut_coop_partition_ids(...)[l]), so
 * the N ranks together hold one copy — and each partition may be any allocation kind, e.g. the
 * paper's managed memory (ut_create UT_ALLOC_MANAGED), which is process-private and so cannot be
 * one shared table. rows: rows of the whole table; part->row_bytes is the
 * row size; part must have >= ut_coop_partition_ids(rows, rb, world, rank, NULL, 0) rows. Every
 * rank of the group must use the same form. NULL on failure. */
UT_API ut_coop* ut_coop_create_partitioned(const ut_table* part, uint64_t rows, int world,
                                           int rank, uint64_t max_n);

/* Host function (no CUDA call): the number of local rows of rank `rank`'s partition (blocks it
 * owns, the last one padded) and, when ids != NULL and cap >= that number, the table row of
 * each local row (ids[l], -1 for the padding). 0 for invalid arguments. */
UT_API uint64_t ut_coop_partition_ids(uint64_t rows, uint64_t row_bytes, int world, int rank,
                                      int64_t* ids, uint64_t cap);

/* Write the CUDA IPC handle (UT_COOP_HANDLE_BYTES bytes) of this rank's region to handle_out and
 * its size to *region_bytes (may be NULL). Returns UT_OK, UT_EINVAL or UT_ECUDA. */
UT_API int ut_coop_export(const ut_coop* c, void* handle_out, uint64_t* region_bytes);

/* Map every other rank's region: handles = world x UT_COOP_HANDLE_BYTES bytes in rank order
 * (this rank's entry is ignored). Returns UT_OK, UT_EINVAL or UT_ECUDA. */
UT_API int ut_coop_open(ut_coop* c, const void* handles);

/* In-process form of ut_coop_open, for one process driving several GPUs with one host thread
 * each (bench.py's box harness over ONE shared table): peers[q] is rank q's handle
 * (peers[rank] == c), every one created in this process with the same world, max_n, table shape
 * and form. Peer regions are addressed directly through unified addressing; peer access is
 * enabled from c's device to each other rank's device (NVLink / NVSwitch P2P; ranks on the same
 * device share its memory). Call on every rank, with c's device current, before the first step.
 * Forward progress: ranks wait for each other on the device, so nothing a step launches may
 * need the device idle. This call loads every kernel of a step (lazy module loading would
 * otherwise load them while a peer's stream waits at a barrier); kernels the CALLER launches
 * between steps must be loaded before the first step too (or run the process with
 * CUDA_MODULE_LOADING=EAGER). Several ranks on ONE device additionally need a hardware queue
 * each (CUDA_DEVICE_MAX_CONNECTIONS >= streams in use, e.g. 32), or a waiting stream can hold the
 * queue its peer's flag write sits in.
 * Returns UT_OK, UT_EINVAL (NULL handle, ranks or layouts disagree) or UT_ENOTSUP (two devices
 * without peer access). */
UT_API int ut_coop_open_local(ut_coop* c, ut_coop* const* peers, int world);

/* Phase 1: send idx_dev[0..n) (device memory, int64, caller-owned, n <= max_n) to the owners.
 * Starts a new step. Asynchronous on `stream`. Returns UT_OK, UT_EINVAL or UT_ECUDA. */
UT_API int ut_coop_dispatch(ut_coop* c, const int64_t* idx_dev, uint64_t n, ut_stream_t stream);

/* Phase 2 (after every rank's phase 1 completed): deduplicate the requests this rank owns and
 * gather the unique rows from host memory into its staging rows. Asynchronous on `stream`. */
UT_API int ut_coop_fetch(ut_coop* c, ut_stream_t stream);

/* Phase 3 (after every rank's phase 2 completed): out_dev[i*rb ..) = row idx[i] of this step's
 * dispatch (>= n*rb bytes of device memory, any alignment). Asynchronous on `stream`. */
UT_API int ut_coop_combine(ut_coop* c, void* out_dev, ut_stream_t stream);

/* The three phases with device-side barriers between them (every rank calls it for the step).
 * Returns UT_OK, UT_EINVAL, UT_ENOTSUP (no stream memory operations) or UT_ECUDA. On UT_EINVAL
 * for n > max_n or a NULL buffer, the rank still took part in the step with n = 0 (its peers'
 * device waits are satisfied); out_dev is untouched. A failure inside the fetch phase still
 * writes this rank's barrier-1 flags. Any other failure before barrier 0 — the wrong current
 * device, unopened peers, a launch error of the dispatch (a broken context) — returns without
 * joining the step: its peers' streams then wait at barrier 0 until the process (or the whole
 * job) is torn down. This is deliberate — joining the step without having dispatched would let
 * the peers combine stale rows from this rank's staging silently — so a rank that sees such an
 * error must abort the job rather than continue. */
UT_API int ut_coop_gather(ut_coop* c, const int64_t* idx_dev, uint64_t n, void* out_dev,
                          ut_stream_t stream);

typedef struct ut_coop_stats {
  uint64_t steps;                /* steps dispatched by this rank                                */
  uint64_t requested_rows;       /* sum of this rank's n                                         */
  uint64_t owner_requests;       /* requests this rank received as an owner (all sources)        */
  uint64_t unique_rows_fetched;  /* rows this rank fetched from host memory as an owner          */
  uint64_t last_unique_rows;     /* ... in the last fetch                                        */
  uint64_t kernel_launches;      /* kernels enqueued by coop calls (the host fetch's gather
                                    kernels are counted by the table's ut_get_stats)             */
  uint64_t stream_memops;        /* flag writes / waits of ut_coop_gather's device barriers      */
  uint64_t block_rows;           /* rows per ownership block                                     */
  uint64_t region_bytes;         /* bytes of this rank's symmetric region                        */
} ut_coop_stats;

/* Fill *s (synchronises with the device for the device-side counters). */
UT_API int ut_coop_get_stats(const ut_coop* c, ut_coop_stats* s);

/* As ut_error_pos, for indices this rank dispatched: syncs `stream`, reports and clears the
 * smallest bad position (-1 and UT_OK if none, UT_ERANGE otherwise). */
UT_API int ut_coop_error_pos(const ut_coop* c, ut_stream_t stream, int64_t* first_bad);

/* Ownership (host function, no CUDA call): the rank owning row id of a rows x row_bytes table
 * split among `world` ranks, and its dense index in the owner's tag table (*local, may be NULL).
 * Blocks of R = 2 MiB / row_bytes rows (one translation region; fewer when the table has under
 * 64 blocks per rank, at least 1) go round-robin: owner = (id / R) mod world. UINT32_MAX for
 * invalid arguments or an id outside [0, rows). */
UT_API uint32_t ut_coop_owner(uint64_t rows, uint64_t row_bytes, int world, int64_t id,
                              uint64_t* local);

/* Release: waits for the device, unmaps the peers' regions, frees this rank's. NULL is a no-op.
 * Every rank should release only after all ranks finished their last step. */
UT_API int ut_coop_release(ut_coop* c);

#ifdef __cplusplus
}
#endif

#endif /* UT_H */
