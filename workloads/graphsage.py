"""GraphSAGE-shaped minibatch index lists over an implicit Chung-Lu power-law graph.

The paper's end-to-end workload is DGL GraphSAGE/GAT minibatch training:
"CPUs need to generate subgraphs for each mini-batch and constantly traverse input graphs to
identify neighboring nodes", and the gather then fetches the features of every
node of the sampled subgraph (Listing 1/2 ``features[neighbor_id]``).
Sampling is NOT on the measured path (it happens on the CPU before the gather);
this module only produces the ``neighbor_id`` lists with the right shape: sizes, duplicate
structure and hub skew. It contains no gather arithmetic.

Graph recipe (nothing is stored, so the 111M-node papers shape costs no RAM):
  * node ranks k in [0, N) carry Chung-Lu weights w_k = (k+1)^-theta, theta = 1/(gamma-1);
  * node id of rank k is perm(k) = (k*A + B) mod N with gcd(A, N) = 1 (hubs spread over ids);
  * deg(v) = max(1, round(E * w_rank(v) / W)), W = sum_k w_k (closed-form approximation);
  * neighbour slot j of v is the node of rank F^-1(u), u = U01(h(seed, v, j)), F the continuous
    CDF of the weights, so neighbours are drawn proportionally to weight (Chung-Lu);
  * a minibatch's roots are batch-size consecutive positions of a second seeded permutation;
  * hop h samples min(deg(v), fanout[h]) distinct slots of every frontier node (stratified
    positions, DGL samples without replacement), hop 0 at the roots (reading R10);
  * the index list is the union of roots and all sampled nodes in first-appearance order
    (DGL's input nodes, reading R11), int64.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

PHI = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _splitmix(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + PHI
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _u01(x: np.ndarray) -> np.ndarray:
    return (x >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


def _coprime_multiplier(n: int, seed: int) -> int:
    a = (int(_splitmix(np.array([seed], dtype=np.uint64))[0]) % n) | 1
    while math.gcd(a, n) != 1:
        a += 2
    return a % n if n > 1 else 0


@dataclass
class ChungLuGraph:
    """Implicit power-law graph: N nodes, about E directed in-edges (reading R12)."""

    n_nodes: int
    n_edges: int
    seed: int = 1
    gamma: float = 2.5
    _a: int = field(init=False)
    _b: int = field(init=False)
    _ainv: int = field(init=False)

    def __post_init__(self):
        n = self.n_nodes
        self.theta = 1.0 / (self.gamma - 1.0)
        self._a = _coprime_multiplier(n, self.seed ^ 0x1234) if n > 1 else 0
        self._b = int(_splitmix(np.array([self.seed ^ 0x5678], dtype=np.uint64))[0]) % n
        self._ainv = pow(self._a, -1, n) if n > 1 else 0
        one = 1.0 - self.theta
        # W = sum_{k=0}^{N-1} (k+1)^-theta ~ integral from 0.5 to N+0.5 of x^-theta dx
        self._w_total = ((n + 0.5) ** one - 0.5 ** one) / one
        self._cdf_hi = (n + 1.0) ** one - 1.0

    # rank <-> node id
    def node_of_rank(self, k: np.ndarray) -> np.ndarray:
        k = k.astype(np.uint64)
        with np.errstate(over="ignore"):
            return ((k * np.uint64(self._a) + np.uint64(self._b)) % np.uint64(self.n_nodes)).astype(np.int64)

    def rank_of_node(self, v: np.ndarray) -> np.ndarray:
        n = np.uint64(self.n_nodes)
        v = v.astype(np.uint64)
        with np.errstate(over="ignore"):
            d = (v + n - np.uint64(self._b)) % n
            # d * ainv may exceed 2^64 for n > 2^32; all configs here have n < 2^27
            return ((d * np.uint64(self._ainv)) % n).astype(np.int64)

    def degree(self, v: np.ndarray) -> np.ndarray:
        k = self.rank_of_node(v).astype(np.float64)
        d = np.rint(self.n_edges * (k + 1.0) ** (-self.theta) / self._w_total)
        return np.maximum(d, 1.0).astype(np.int64)

    def neighbour(self, v: np.ndarray, slot: np.ndarray) -> np.ndarray:
        """Node at neighbour slot `slot` of node `v` (arrays of equal length)."""
        with np.errstate(over="ignore"):
            h = _splitmix(np.uint64(self.seed) ^ (v.astype(np.uint64) * PHI + slot.astype(np.uint64)))
            h = _splitmix(h)
        u = _u01(h)
        one = 1.0 - self.theta
        x = (1.0 + u * self._cdf_hi) ** (1.0 / one) - 1.0
        rank = np.minimum(np.floor(x), self.n_nodes - 1).astype(np.int64)
        return self.node_of_rank(rank)


def _first_appearance_unique(a: np.ndarray) -> np.ndarray:
    _, first = np.unique(a, return_index=True)
    return a[np.sort(first)]


@dataclass
class GraphSageSampler:
    """Per-rank minibatch index lists: roots partitioned by rank, fanout per hop."""

    graph: ChungLuGraph
    batch_size: int
    fanouts: tuple
    seed: int = 7
    reverse_fanouts: bool = False

    def __post_init__(self):
        n = self.graph.n_nodes
        self._ra = _coprime_multiplier(n, self.seed ^ 0x9ABC)
        self._rb = int(_splitmix(np.array([self.seed ^ 0xDEF0], dtype=np.uint64))[0]) % n

    def roots(self, batch: int, rank: int = 0, world: int = 1) -> np.ndarray:
        n = self.graph.n_nodes
        start = (batch * world + rank) * self.batch_size
        p = (np.arange(start, start + self.batch_size, dtype=np.uint64)) % np.uint64(n)
        with np.errstate(over="ignore"):
            r = (p * np.uint64(self._ra) + np.uint64(self._rb)) % np.uint64(n)
        return _first_appearance_unique(r.astype(np.int64))

    def minibatch(self, batch: int, rank: int = 0, world: int = 1) -> np.ndarray:
        """The int64 ``neighbor_id`` list of one minibatch (roots first, then new nodes by hop)."""
        fan = tuple(reversed(self.fanouts)) if self.reverse_fanouts else tuple(self.fanouts)
        nodes = self.roots(batch, rank, world)
        frontier = nodes
        bkey = np.uint64((self.seed * 1000003 + batch * 8191 + rank * 131) & 0xFFFFFFFFFFFFFFFF)
        for hop, f in enumerate(fan):
            deg = self.graph.degree(frontier)
            cnt = np.minimum(deg, f)
            total = int(cnt.sum())
            owner = np.repeat(np.arange(frontier.size), cnt)
            t = np.arange(total, dtype=np.int64) - np.repeat(np.cumsum(cnt) - cnt, cnt)
            v = frontier[owner]
            with np.errstate(over="ignore"):
                h = _splitmix(bkey ^ (np.uint64(hop + 1) * PHI) ^ (v.astype(np.uint64) * _M1 + t.astype(np.uint64)))
            u = _u01(h)
            d = deg[owner].astype(np.float64)
            c = cnt[owner].astype(np.float64)
            slot = np.minimum(np.floor((t + u) * d / c), d - 1).astype(np.int64)
            nbr = self.graph.neighbour(v, slot)
            merged = _first_appearance_unique(np.concatenate([frontier, nbr]))
            frontier = merged
            nodes = _first_appearance_unique(np.concatenate([nodes, merged]))
        return nodes


# Paper-shaped configs (Table 4; BASELINE.json configs).
CONFIGS = {
    "reddit": dict(n_nodes=232_965, n_edges=11_600_000, row_bytes=602 * 4, batch=1000,
                   fanouts=(25, 10)),
    "products": dict(n_nodes=2_449_029, n_edges=61_900_000, row_bytes=100 * 4, batch=1024,
                     fanouts=(15, 10, 5)),
    "papers": dict(n_nodes=111_000_000, n_edges=1_600_000_000, row_bytes=128 * 4, batch=1024,
                   fanouts=(15, 10, 5)),
}


def sampler_for(config: str, seed: int = 1, reverse_fanouts: bool = False,
                edges: int | None = None) -> GraphSageSampler:
    """The config's sampler; `edges` overrides Table 4's E (reddit's E = 114.6M
    sensitivity run, the paper does not say whether its E counts directed edges)."""
    c = CONFIGS[config]
    g = ChungLuGraph(c["n_nodes"], edges or c["n_edges"], seed=seed)
    return GraphSageSampler(g, c["batch"], c["fanouts"], seed=seed + 6,
                            reverse_fanouts=reverse_fanouts)


def minibatch_job(args) -> np.ndarray:
    """Picklable worker: (config, seed, batch, rank, world, reverse[, edges]) -> index list."""
    config, seed, batch, rank, world, reverse = args[:6]
    edges = args[6] if len(args) > 6 else None
    return sampler_for(config, seed=seed, reverse_fanouts=reverse, edges=edges).minibatch(batch, rank, world)
