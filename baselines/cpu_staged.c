/*
 * baselines/cpu_staged.c — the paper's CPU-centric baseline ("Py", Fig. 2a),
 * reported beside the GPU gather for context (BASELINE.json north_star). Not on the product path.
 *
 * The CPU gathers the rows into cache (1) and writes them to a temporary contiguous buffer (2)
 * with several threads ("the data gathering part of the code is multithreaded"); the
 * caller then issues one DMA of that buffer to the GPU (3)(4) (cudaMemcpyAsync from pinned
 * staging, Listing 1 `features[neighbor_id].to("cuda")`).
 */
#include <stdint.h>
#include <string.h>
#include <omp.h>

void cpu_staged_gather(const uint8_t* table, uint64_t rb, const int64_t* idx, uint64_t n,
                       uint8_t* staging, int threads)
{
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(static, 256) num_threads(nt)
    for (int64_t i = 0; i < (int64_t)n; ++i)
        memcpy(staging + (uint64_t)i * rb, table + (uint64_t)idx[i] * rb, rb);
}

/* Host DRAM read bandwidth probe for the per-box roofline (min(R_concurrent, R_dram), SURVEY
 * §8d): all threads stream-read [p, p+bytes) with 64-bit loads; returns a checksum so the reads
 * are not elided. */
uint64_t host_read_sum(const uint8_t* p, uint64_t bytes, int threads)
{
    int nt = threads > 0 ? threads : omp_get_max_threads();
    const uint64_t* q = (const uint64_t*)p;
    int64_t words = (int64_t)(bytes / 8);
    uint64_t acc = 0;
#pragma omp parallel for schedule(static) num_threads(nt) reduction(^:acc)
    for (int64_t i = 0; i < words; ++i) acc ^= q[i];
    return acc;
}
