"""Pins of the sampling oracle (oracle/ut_oracle_sample.c) against closed forms:
SPEC's K5 / star examples, breadth-first order when the fanout covers every
degree (a textbook BFS), and the stratified without-replacement slot structure decoded from a
tree whose child ids encode their slot."""
import collections

import numpy as np
import pytest

import oracle


class CSR:
    def __init__(self, adj):
        self.n = len(adj)
        self.indptr = np.zeros(self.n + 1, dtype=np.int64)
        for v, a in enumerate(adj):
            self.indptr[v + 1] = self.indptr[v] + len(a)
        self.indices = np.array([u for a in adj for u in a] or [0], dtype=np.int32)

    def sample(self, seeds, fanouts, seed=1):
        return oracle.sample(self.indptr.ctypes.data, self.indices.ctypes.data, self.n, seeds,
                             fanouts, seed).tolist()


def bfs_order(adj, seeds, hops):
    seen, order = set(), []
    q = collections.deque()
    for s in seeds:
        if s not in seen:
            seen.add(s)
            order.append(s)
            q.append((s, 0))
    while q:
        v, d = q.popleft()
        if d == hops:
            continue
        for u in adj[v]:
            if u not in seen:
                seen.add(u)
                order.append(u)
                q.append((u, d + 1))
    return order


def test_k5_fanout_2_gives_3_nodes():
    adj = [[u for u in range(5) if u != v] for v in range(5)]
    g = CSR(adj)
    for s in range(20):
        out = g.sample([0], [2], seed=s)
        assert len(out) == 3 and out[0] == 0 and len(set(out)) == 3


def test_star_full_fanout_in_adjacency_order():
    adj = [list(range(1, 8))] + [[0]] * 7
    g = CSR(adj)
    assert g.sample([0], [7]) == list(range(8))
    assert g.sample([0], [100]) == list(range(8))
    assert g.sample([3], [5, 7]) == [3, 0, 1, 2, 4, 5, 6, 7]


@pytest.mark.parametrize("trial", range(8))
def test_full_fanout_equals_bfs(trial):
    rng = np.random.default_rng(trial)
    n = int(rng.integers(5, 60))
    adj = [sorted(set(rng.integers(0, n, size=int(rng.integers(0, 6))).tolist())) for _ in range(n)]
    g = CSR(adj)
    seeds = rng.integers(0, n, size=int(rng.integers(1, 5))).tolist()
    hops = int(rng.integers(1, 4))
    assert g.sample(seeds, [1000] * hops, seed=trial) == bfs_order(adj, seeds, hops)


def test_stratified_slots_without_replacement():
    """Tree: node v (< 500 roots) has D children v*D + 500 + slot. One hop with fanout f < D
    samples exactly f children per root, one per stratum [floor(tD/f), floor((t+1)D/f))."""
    R, D = 500, 23
    adj = [[R + v * D + s for s in range(D)] for v in range(R)] + [[] for _ in range(R * D)]
    g = CSR(adj)
    for f in (1, 2, 5, 22):
        out = g.sample(list(range(R)), [f], seed=f)
        assert out[:R] == list(range(R))
        kids = out[R:]
        assert len(kids) == R * f
        hist = np.zeros(D, dtype=np.int64)
        for k, c in enumerate(kids):
            v, t = k // f, k % f
            slot = c - R - v * D
            assert 0 <= slot < D and (c - R) // D == v
            assert t * D // f <= slot < (t + 1) * D // f
            hist[slot] += 1
        if f == 1:   # one stratum covering all slots: roughly uniform
            assert hist.min() > 0 and hist.max() < 3 * R / D


def test_deterministic_and_seed_sensitive():
    rng = np.random.default_rng(5)
    n = 3000
    adj = [sorted(set(rng.integers(0, n, size=40).tolist())) for _ in range(n)]
    g = CSR(adj)
    a = g.sample([1, 2, 3], [5, 3], seed=11)
    assert a == g.sample([1, 2, 3], [5, 3], seed=11)
    assert a != g.sample([1, 2, 3], [5, 3], seed=12)
    assert len(a) == len(set(a)) and a[:3] == [1, 2, 3]


def test_duplicate_seeds_and_bad_seed():
    adj = [[1], [0], []]
    g = CSR(adj)
    assert g.sample([1, 1, 0], [1]) == [1, 0]
    with pytest.raises(ValueError):
        g.sample([3], [1])
