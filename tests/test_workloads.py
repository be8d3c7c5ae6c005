"""Input generators: determinism, ranges, the guard page, GraphSAGE list structure."""
import os
import subprocess
import sys

import numpy as np

import workloads
from workloads import graphsage as gs


def test_table_fill_deterministic_and_self_identifying():
    rows, rb = 5000, 37
    a = np.empty(rows * rb, np.uint8)
    b = np.empty(rows * rb, np.uint8)
    workloads.fill_table(a, rows, rb, 99, threads=1)
    workloads.fill_table(b, rows, rb, 99, threads=4)
    assert a.tobytes() == b.tobytes()
    np.testing.assert_array_equal(workloads.decode_row_ids(a, rb), np.arange(rows))
    assert len({a[i * rb:(i + 1) * rb].tobytes() for i in range(rows)}) == rows
    c = np.empty(rows * rb, np.uint8)
    workloads.fill_table(c, rows, rb, 100)
    assert c.tobytes() != a.tobytes()


def test_narrow_rows_encode_low_id_bytes():
    rows, rb = 70000, 2
    a = np.empty(rows * rb, np.uint8)
    workloads.fill_table(a, rows, rb, 1)
    np.testing.assert_array_equal(workloads.decode_row_ids(a, rb), np.arange(rows) & 0xFFFF)


def test_uniform_idx():
    x = workloads.uniform_idx(200_000, 1000, 5)
    assert x.dtype == np.int64 and x.min() >= 0 and x.max() < 1000
    np.testing.assert_array_equal(x, workloads.uniform_idx(200_000, 1000, 5))
    h = np.bincount(x, minlength=1000)
    assert h.min() > 120 and h.max() < 290
    big = workloads.uniform_idx(100_000, 1 << 32, 1)
    assert big.max() >= (1 << 31)      # int64 ids beyond int32 range (reading R2)


def test_guard_page_faults_past_the_end():
    code = (
        "import ctypes, workloads\n"
        "hb = workloads.HostBuffer(1000, kind='guarded')\n"
        "assert (hb.addr + 1000) % 4096 == 0\n"
        "ctypes.c_uint8.from_address(hb.addr + 999).value\n"
        "print('last-byte-ok', flush=True)\n"
        "ctypes.c_uint8.from_address(hb.addr + 1000).value\n"
        "print('NO-FAULT')\n"
    )
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True)
    assert "last-byte-ok" in p.stdout
    assert "NO-FAULT" not in p.stdout and p.returncode != 0


def test_shm_buffer_shared_between_mappings():
    name = f"ut_test_{os.getpid()}"
    a = workloads.HostBuffer(4096, kind="shm", name=name, create=True)
    try:
        a.array()[:4] = [1, 2, 3, 4]
        b = workloads.HostBuffer(4096, kind="shm", name=name, create=False)
        assert list(b.array()[:4]) == [1, 2, 3, 4]
        b.close()
    finally:
        a.close(unlink=True)


def test_graph_degrees_match_edge_budget():
    g = gs.ChungLuGraph(100_000, 2_000_000, seed=3)
    d = g.degree(np.arange(100_000))
    assert abs(d.sum() / 2_000_000 - 1) < 0.05
    assert d.max() > 50 * d.mean()                    # power-law hubs
    ranks = g.rank_of_node(g.node_of_rank(np.arange(100_000)))
    np.testing.assert_array_equal(ranks, np.arange(100_000))


def test_minibatch_structure():
    s = gs.GraphSageSampler(gs.ChungLuGraph(50_000, 1_000_000, seed=2), 64, (5, 3), seed=4)
    a = s.minibatch(0)
    np.testing.assert_array_equal(a, s.minibatch(0))
    assert a.dtype == np.int64 and len(np.unique(a)) == a.size
    assert a.min() >= 0 and a.max() < 50_000
    roots = s.roots(0)
    np.testing.assert_array_equal(a[:roots.size], roots)
    assert roots.size <= a.size <= roots.size * (1 + 5 + 5 * 3 + 5 * 3)
    r0 = set(s.roots(0, rank=0, world=2))
    r1 = set(s.roots(0, rank=1, world=2))
    assert not (r0 & r1)


def test_fill_table_on_pinned_threads_matches_fill_table():
    """The per-node fill (one thread pinned per CPU, first touch on that node) writes exactly the
    table fill_table writes, for any thread count and a ragged last slice."""
    rows, rb = 1001, 68
    a = np.zeros(rows * rb, np.uint8)
    workloads.fill_table(a, rows, rb, 9)
    cpus = workloads.node_cpus(0) or [0]
    for k in (1, 3, len(cpus)):
        b = np.zeros(rows * rb, np.uint8)
        assert workloads.fill_table_on(b, rows, rb, 9, (cpus * 3)[:k])
        assert b.tobytes() == a.tobytes()
