/*
 * oracle/ut_oracle_sample.c — TEST INFRASTRUCTURE ONLY (same rules as ut_oracle.c).
 *
 * Plain CPU definition of multi-hop neighbour sampling over a CSR graph: the step
 * before the gather, which the paper leaves on the CPU ("CPUs need to generate subgraphs for each
 * mini-batch and constantly traverse input graphs to identify neighboring nodes", PAPER.md:95;
 * DGL GraphSAGE sampling). Semantics (reading R17):
 *   frontier_0 = seeds (first-appearance unique);
 *   hop h (fanout f_h): for every node v of frontier_h in order, with deg = indptr[v+1]-indptr[v]:
 *     deg <= f_h: take neighbour slots 0..deg-1;
 *     deg >  f_h: take one slot per stratum t < f_h: lo = floor(t*deg/f_h), hi = floor((t+1)*deg/f_h),
 *                 slot = lo + H(seed, h, v, t) mod (hi - lo)   (distinct slots, sampling without
 *                 replacement as DGL does);
 *     candidates = the neighbours at those slots, in (v, t) order;
 *   frontier_{h+1} = frontier_h followed by the candidates not yet in it, first appearance first;
 *   the minibatch node list is the last frontier (= the union of all hops, seeds first).
 *   H(seed, h, v, t) = m(m(m(seed + (h+1)*PHI) ^ v) + t), m = SplitMix64 finaliser.
 * Every membership test is a plain byte flag per node; no hashing, no sorting.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define PHI 0x9E3779B97F4A7C15ull

static uint64_t m64(uint64_t x)
{
    uint64_t z = x + PHI;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t oracle_sample_hash(uint64_t seed, uint64_t hop, uint64_t v, uint64_t t)
{
    return m64(m64(m64(seed + (hop + 1) * PHI) ^ v) + t);
}

/* Returns the node count (<= cap, written to out), -1 if cap is too small (count in *need),
 * -2 if a seed is out of [0, n_nodes), -3 on allocation failure. */
int64_t oracle_sample(const int64_t* indptr, const int32_t* indices, uint64_t n_nodes,
                      const int64_t* seeds, uint64_t n_seeds, const int32_t* fanouts, int hops,
                      uint64_t seed, int64_t* out, uint64_t cap, uint64_t* need)
{
    uint8_t* in_front = calloc(n_nodes ? n_nodes : 1, 1);
    uint64_t size = 0, alloc = n_seeds + 16;
    int64_t* front = malloc(alloc * sizeof(int64_t));
    if (!in_front || !front) { free(in_front); free(front); return -3; }
    for (uint64_t i = 0; i < n_seeds; ++i) {
        int64_t v = seeds[i];
        if (v < 0 || (uint64_t)v >= n_nodes) { free(in_front); free(front); return -2; }
        if (!in_front[v]) { in_front[v] = 1; front[size++] = v; }
    }
    for (int h = 0; h < hops; ++h) {
        const uint64_t f = (uint64_t)fanouts[h];
        const uint64_t old = size;            /* nodes expanded at this hop: frontier_h */
        for (uint64_t i = 0; i < old; ++i) {
            const int64_t v = front[i];
            const uint64_t base = (uint64_t)indptr[v];
            const uint64_t deg = (uint64_t)(indptr[v + 1] - indptr[v]);
            const uint64_t cnt = deg < f ? deg : f;
            for (uint64_t t = 0; t < cnt; ++t) {
                uint64_t slot = t;
                if (deg > f) {
                    const uint64_t lo = t * deg / f, hi = (t + 1) * deg / f;
                    slot = lo + oracle_sample_hash(seed, (uint64_t)h, (uint64_t)v, t) % (hi - lo);
                }
                const int64_t c = indices[base + slot];
                if (in_front[c]) continue;
                in_front[c] = 1;
                if (size == alloc) {
                    alloc *= 2;
                    int64_t* g = realloc(front, alloc * sizeof(int64_t));
                    if (!g) { free(in_front); free(front); return -3; }
                    front = g;
                }
                front[size++] = c;
            }
        }
    }
    if (need) *need = size;
    int64_t rc = -1;
    if (size <= cap) {
        memcpy(out, front, size * sizeof(int64_t));
        rc = (int64_t)size;
    }
    free(in_front);
    free(front);
    return rc;
}
