/*
 * oracle/ut_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously correct CPU definition of what the unified-tensor gather computes.
 * Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and --impl reference)
 * may load this file's library. It shares no code, header, table or helper with the CUDA path
 * (paper_2101_07956_b200/csrc/) and includes nothing from it.
 *
 * Definition followed (PAPER.md, cited by line):
 *   - The feature table is "a 2D array where the row indices are the IDs of nodes and the
 *     columns are the features of each node" (§2.2).
 *   - `unified_tensor[gpu_tensor]`: "Indexing unified tensor with GPU tensor" (Table 1);
 *     Listing 2 `input_features = features[neighbor_id]`: output row i is the
 *     feature row of node neighbor_id[i], in order ("the first 11 threads access the 11 features
 *     of the 0th node, next 11 threads access the 11 features of the 2nd node").
 *   - The alignment optimisation does not change the result: "the output indices are also
 *     identically adjusted to maintain the ordering".
 * Readings where the paper is silent: rows are copied as bytes (R3);
 * indices are int64 (R2); an index < 0 or >= rows zero-fills its output row and the smallest
 * such position is reported (R4, after SPEC.md:151 "index error naming the offending position");
 * n == 0 produces nothing (R5).
 */
#include <stdint.h>
#include <string.h>

/* out[i*rb .. (i+1)*rb) = table[idx[i]*rb .. (idx[i]+1)*rb) for i in [0, n).
 * Returns the smallest i with idx[i] out of [0, rows), or -1 if every index is in range. */
int64_t oracle_gather(const uint8_t* table, uint64_t rows, uint64_t rb,
                      const int64_t* idx, uint64_t n, uint8_t* out)
{
    int64_t first_bad = -1;
    for (uint64_t i = 0; i < n; ++i) {
        int64_t r = idx[i];
        if (r < 0 || (uint64_t)r >= rows) {
            if (first_bad < 0) first_bad = (int64_t)i;
            memset(out + i * rb, 0, rb);
            continue;
        }
        memcpy(out + i * rb, table + (uint64_t)r * rb, rb);
    }
    return first_bad;
}
