/*
 * workloads/gen.c — seeded synthetic INPUT generators (no gather arithmetic).
 *
 * Shared by the tests, the oracle side and the CUDA side as the source of inputs only: it
 * fills the host feature table (whole, or the sub-table of chosen row ids, gen_fill_rows) and
 * draws uniform index lists. It copies no rows: every row it writes is computed from its id and
 * the seed, the table's definition. It is never the source of an expected gather result — those
 * come from oracle/ only (bench builds a sub-table here and gathers from it with the oracle).
 *
 * Recipe:
 *   splitmix64(x): the standard SplitMix64 finaliser.
 *   Table content ("self-identifying"): byte b of row r is byte (b mod 8) of
 *       splitmix64(seed ^ (r * PHI + b / 8)),
 *   except that the first min(rb, 8) bytes of row r are r's little-endian bytes, so that any
 *   fetched row decodes to the row id it came from and no two rows are equal.
 *   Uniform indices: idx[i] = floor(splitmix64(seed ^ (i * PHI)) * rows / 2^64)
 *   (uniform with replacement over [0, rows), reading R9).
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <sched.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <omp.h>

#define PHI 0x9E3779B97F4A7C15ull

static inline uint64_t splitmix64(uint64_t x)
{
    uint64_t z = x + PHI;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t gen_splitmix64(uint64_t x) { return splitmix64(x); }

static inline void fill_row(uint8_t* row, uint64_t r, uint64_t rb, uint64_t seed)
{
    uint64_t base = r * PHI;
    uint64_t b = 0;
    for (; b + 8 <= rb; b += 8) {
        uint64_t w = splitmix64(seed ^ (base + b / 8));
        memcpy(row + b, &w, 8);
    }
    if (b < rb) {
        uint64_t w = splitmix64(seed ^ (base + b / 8));
        memcpy(row + b, &w, rb - b);
    }
    memcpy(row, &r, rb < 8 ? rb : 8);
}

/* Fill rows*rb bytes at dst with the self-identifying content. Rows are independent, so the
 * loop is split over `threads` OpenMP threads (threads <= 0: all available). */
void gen_fill_table(uint8_t* dst, uint64_t rows, uint64_t rb, uint64_t seed, int threads)
{
    int64_t R = (int64_t)rows;
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(static, 4096) num_threads(nt)
    for (int64_t r = 0; r < R; ++r)
        fill_row(dst + (uint64_t)r * rb, (uint64_t)r, rb, seed);
}

/* The same content, written by one thread pinned to each of cpus[0..ncpus) (each a contiguous
 * slice of rows), so that the pages are first touched -- and, under the default first-touch
 * policy, placed -- on those CPUs' NUMA node (bench.py --numa replica: one replica per node).
 * Returns 0, or -1 if a thread could not be started or pinned. */
struct fill_part { uint8_t* dst; uint64_t lo, hi, rb, seed; int cpu, rc; };

static void* fill_part_run(void* p)
{
    struct fill_part* f = (struct fill_part*)p;
    cpu_set_t set;
    CPU_ZERO(&set);
    CPU_SET(f->cpu, &set);
    f->rc = pthread_setaffinity_np(pthread_self(), sizeof set, &set) == 0 ? 0 : -1;
    for (uint64_t r = f->lo; r < f->hi; ++r)
        fill_row(f->dst + r * f->rb, r, f->rb, f->seed);
    return NULL;
}

int gen_fill_table_on(uint8_t* dst, uint64_t rows, uint64_t rb, uint64_t seed, const int* cpus, int ncpus)
{
    if (ncpus < 1) return -1;
    struct fill_part* parts = (struct fill_part*)calloc((size_t)ncpus, sizeof *parts);
    pthread_t* th = (pthread_t*)calloc((size_t)ncpus, sizeof *th);
    int rc = parts && th ? 0 : -1;
    int started = 0;
    const uint64_t per = (rows + (uint64_t)ncpus - 1) / (uint64_t)ncpus;
    for (int i = 0; rc == 0 && i < ncpus; ++i) {
        uint64_t lo = (uint64_t)i * per, hi = lo + per;
        if (lo > rows) lo = rows;
        if (hi > rows) hi = rows;
        parts[i] = (struct fill_part){dst, lo, hi, rb, seed, cpus[i], 0};
        if (pthread_create(&th[i], NULL, fill_part_run, &parts[i]) != 0) rc = -1;
        else ++started;
    }
    for (int i = 0; i < started; ++i) {
        pthread_join(th[i], NULL);
        if (parts[i].rc != 0) rc = -1;
    }
    if (rc != 0 && started < ncpus)      /* finish the rows of threads that never started */
        gen_fill_table(dst, rows, rb, seed, 0);
    free(parts);
    free(th);
    return rc;
}

/* Row k of dst = the self-identifying content of table row ids[k] (as gen_fill_table writes it);
 * ids[k] < 0 gives a zero row. Fills a partition of a table or a sub-table of chosen rows
 * (table input, not an expected gather result). */
void gen_fill_rows(uint8_t* dst, const int64_t* ids, uint64_t n, uint64_t rb, uint64_t seed, int threads)
{
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(static, 4096) num_threads(nt)
    for (int64_t k = 0; k < (int64_t)n; ++k) {
        uint8_t* row = dst + (uint64_t)k * rb;
        if (ids[k] < 0) {
            memset(row, 0, rb);
            continue;
        }
        uint64_t r = (uint64_t)ids[k];
        uint64_t base = r * PHI;
        uint64_t b = 0;
        for (; b + 8 <= rb; b += 8) {
            uint64_t w = splitmix64(seed ^ (base + b / 8));
            memcpy(row + b, &w, 8);
        }
        if (b < rb) {
            uint64_t w = splitmix64(seed ^ (base + b / 8));
            memcpy(row + b, &w, rb - b);
        }
        memcpy(row, &r, rb < 8 ? rb : 8);
    }
}

/* idx[i] = floor(splitmix64(seed ^ (i*PHI)) * rows / 2^64), i in [0, n). */
void gen_uniform_idx(int64_t* idx, uint64_t n, uint64_t rows, uint64_t seed)
{
    for (uint64_t i = 0; i < n; ++i) {
        __uint128_t p = (__uint128_t)splitmix64(seed ^ (i * PHI)) * rows;
        idx[i] = (int64_t)(uint64_t)(p >> 64);
    }
}

/* ---- host memory for tables (plain mmap; the library under test pins it itself) ---------- */
#include <sys/mman.h>
#include <unistd.h>

/* Anonymous private mapping of `bytes`, transparent-hugepage advised when hugepage != 0.
 * Returns NULL on failure. */
void* gen_map(uint64_t bytes, int hugepage)
{
    void* p = mmap(NULL, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return NULL;
#ifdef MADV_HUGEPAGE
    if (hugepage) madvise(p, bytes, MADV_HUGEPAGE);
#endif
    return p;
}

int gen_unmap(void* p, uint64_t bytes) { return munmap(p, bytes); }

/* Guard-page layout for over-read tests: [PROT_NONE page][data pages][PROT_NONE page], with the
 * returned pointer placed so that `bytes` end exactly at the start of the trailing guard page.
 * *map_base / *map_len describe the whole mapping for gen_unmap. */
void* gen_map_guarded(uint64_t bytes, void** map_base, uint64_t* map_len)
{
    uint64_t pg = (uint64_t)sysconf(_SC_PAGESIZE);
    uint64_t data = (bytes + pg - 1) / pg * pg;
    uint64_t len = data + 2 * pg;
    uint8_t* p = (uint8_t*)mmap(NULL, len, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
    if (p == MAP_FAILED) return NULL;
    if (mprotect(p, pg, PROT_NONE) != 0 || mprotect(p + pg + data, pg, PROT_NONE) != 0) {
        munmap(p, len);
        return NULL;
    }
    *map_base = p;
    *map_len = len;
    return p + pg + data - bytes;
}

/* ---- explicit CSR graph (for GPU-side sampling) ------------------------------
 * Chung-Lu power law like workloads/graphsage.py, materialised: node of rank k is
 * (k*A + B) mod N; deg(rank k) = max(1, round(E * (k+1)^-theta / W)); neighbour j of node v is
 * the node of rank floor(F^-1(u)), u = U01(splitmix64(seed ^ (v*PHI + j))), F the continuous
 * weight CDF. indptr is int64[N+1], indices int32[indptr[N]]. */
#include <math.h>

static uint64_t gcd_u64(uint64_t a, uint64_t b) { while (b) { uint64_t t = a % b; a = b; b = t; } return a; }

static uint64_t coprime_mult(uint64_t n, uint64_t seed)
{
    uint64_t a = (splitmix64(seed) % n) | 1;
    while (gcd_u64(a, n) != 1) a += 2;
    return a % n;
}

/* Fills indptr[0..N] (int64). Returns the edge count indptr[N]. */
int64_t gen_chunglu_indptr(int64_t* indptr, uint64_t N, uint64_t E, double gamma, uint64_t seed)
{
    const double theta = 1.0 / (gamma - 1.0), one = 1.0 - theta;
    const double W = (pow((double)N + 0.5, one) - pow(0.5, one)) / one;
    const uint64_t A = N > 1 ? coprime_mult(N, seed ^ 0x1234) : 0;
    const uint64_t B = N > 1 ? splitmix64(seed ^ 0x5678) % N : 0;
    for (uint64_t k = 0; k < N; ++k) {
        double d = nearbyint((double)E * pow((double)k + 1.0, -theta) / W);
        int64_t deg = d < 1.0 ? 1 : (int64_t)d;
        uint64_t v = (uint64_t)(((__uint128_t)k * A + B) % N);
        indptr[v + 1] = deg;
    }
    indptr[0] = 0;
    for (uint64_t v = 0; v < N; ++v) indptr[v + 1] += indptr[v];
    return indptr[N];
}

void gen_chunglu_indices(const int64_t* indptr, int32_t* indices, uint64_t N, double gamma,
                         uint64_t seed, int threads)
{
    const double theta = 1.0 / (gamma - 1.0), one = 1.0 - theta;
    const double cdf_hi = pow((double)N + 1.0, one) - 1.0;
    const uint64_t A = N > 1 ? coprime_mult(N, seed ^ 0x1234) : 0;
    const uint64_t B = N > 1 ? splitmix64(seed ^ 0x5678) % N : 0;
    int nt = threads > 0 ? threads : omp_get_max_threads();
#pragma omp parallel for schedule(dynamic, 4096) num_threads(nt)
    for (int64_t v = 0; v < (int64_t)N; ++v) {
        for (int64_t p = indptr[v]; p < indptr[v + 1]; ++p) {
            uint64_t h = splitmix64(splitmix64(seed ^ ((uint64_t)v * PHI + (uint64_t)(p - indptr[v]))));
            double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
            double x = pow(1.0 + u * cdf_hi, 1.0 / one) - 1.0;
            uint64_t rank = x >= (double)(N - 1) ? N - 1 : (uint64_t)x;
            indices[p] = (int32_t)(((__uint128_t)rank * A + B) % N);
        }
    }
}

/* ---- NUMA placement of a table (NUMA-interleaved by default) ------------------
 * mbind(MPOL_INTERLEAVE) over all online nodes before first touch. Returns the number of nodes
 * used (0 when the kernel has no NUMA support or a single node: nothing to do). */
#include <sys/syscall.h>
#include <stdio.h>

int gen_numa_nodes(void)
{
    int n = 0;
    for (int i = 0; i < 1024; ++i) {
        char path[96];
        snprintf(path, sizeof path, "/sys/devices/system/node/node%d", i);
        if (access(path, F_OK) == 0) ++n;
        else if (i > 64 && n) break;
    }
    return n;
}

/* mbind(MPOL_BIND) of [addr, addr+bytes) to one node before first touch. 0 on success. */
int gen_bind_node(void* addr, uint64_t bytes, int node)
{
    if (node < 0 || node >= 1024) return -1;
    unsigned long mask[16] = {0};
    mask[node / 64] |= 1ul << (node % 64);
    return syscall(SYS_mbind, addr, bytes, 2 /* MPOL_BIND */, mask, 1024ul, 0u) == 0 ? 0 : -1;
}

int gen_interleave(void* addr, uint64_t bytes)
{
    int nodes = gen_numa_nodes();
    if (nodes <= 1) return 0;
    unsigned long mask[16] = {0};
    for (int i = 0; i < nodes && i < 1024; ++i) mask[i / 64] |= 1ul << (i % 64);
    long rc = syscall(SYS_mbind, addr, bytes, 3 /* MPOL_INTERLEAVE */, mask, 1024ul, 0u);
    return rc == 0 ? nodes : -1;
}
