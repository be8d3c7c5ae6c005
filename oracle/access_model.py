"""oracle.access_model — TEST INFRASTRUCTURE ONLY: the paper's indexing kernels as access traces.

PAPER.md §4.5 describes two GPU indexing schemes for a unified tensor:

* "PyD Naive" — the stock PyTorch indexing kernel: "each thread accesses a single feature. For
  example, the first 11 threads access the 11 features of the 0th node, next 11 threads access
  the 11 features of the 2nd node, and so on" (Fig. 5): thread t = r*W + j reads
  element rows[r]*W + j and writes output element r*W + j.
* "PyD Optimized" — the circular shift: "all threads calculate the required index offset values
  to make aligned accesses ... the threads need to do a right shift by an offset of 1. The
  threads on the edges check the boundary conditions and make additional adjustments by adding
  or subtracting the length of the node feature ... the output indices are also identically
  adjusted to maintain the ordering" (Fig. 6).

The paper gives no formula for the offset. Reading R13: row r's
shift is s_r = (r*W - rows[r]*W) mod L, L = elements per cacheline, and thread j of row r reads
element rows[r]*W + ((j + s_r) mod W) and writes output element r*W + ((j + s_r) mod W); the mod
W is the "adding or subtracting the length of the node feature" at the edges. A PCIe request is
counted as one distinct (warp, cacheline) pair (reading R14), which is how
"7 to 5" is reproduced.

Everything here is pure-Python loops over small cases; it predicts request counts for the
ablation kernels and is pinned by tests/test_access_model.py.
"""
from __future__ import annotations


def compute_shifts(rows, W: int, L: int) -> list[int]:
    """s_r = (r*W - rows[r]*W) mod L for every output row r (reading R13)."""
    return [((r * W) - (g * W)) % L for r, g in enumerate(rows)]


def naive_trace(rows, W: int) -> list[tuple[int, int, int]]:
    """(thread, source element, output element) of the stock thread-per-element kernel."""
    out = []
    for r, g in enumerate(rows):
        for j in range(W):
            out.append((r * W + j, g * W + j, r * W + j))
    return out


def shifted_trace(rows, W: int, L: int) -> list[tuple[int, int, int]]:
    """(thread, source element, output element) of the circular-shift kernel (reading R13)."""
    shifts = compute_shifts(rows, W, L)
    out = []
    for r, g in enumerate(rows):
        s = shifts[r]
        for j in range(W):
            e = (j + s) % W
            out.append((r * W + j, g * W + e, r * W + e))
    return out


def execute(trace, src_flat, n_out: int) -> list:
    """Run a trace: out[o] = src[e] for every (thread, e, o); returns the output list."""
    out = [None] * n_out
    for _, e, o in trace:
        out[o] = src_flat[e]
    return out


def count_requests(trace, warp: int, line_elems: int, base_elem_offset: int = 0,
                   threads=None) -> int:
    """Distinct (warp, cacheline) pairs over the trace (optionally only the given threads).

    warp: threads per warp; line_elems: elements per cacheline; base_elem_offset: the table's
    start offset inside its first cacheline, in elements."""
    pairs = set()
    for t, e, _ in trace:
        if threads is not None and t not in threads:
            continue
        pairs.add((t // warp, (e + base_elem_offset) // line_elems))
    return len(pairs)


def lines_touched(start_byte: int, nbytes: int, line: int) -> int:
    """Number of `line`-byte lines that bytes [start, start+nbytes) touch (0 if nbytes == 0)."""
    if nbytes == 0:
        return 0
    return (start_byte + nbytes - 1) // line - start_byte // line + 1
