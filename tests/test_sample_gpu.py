"""Parity of GPU-side neighbour sampling (ut_sample) with the sampling oracle:
the node lists must be identical (order included) — integer work, bit-exact bar."""
import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
ut = pytest.importorskip("paper_2101_07956_b200")

pytestmark = pytest.mark.gpu


class HostCSR:
    """CSR arrays in page-aligned buffers of their own: registration pins whole pages, so the
    arrays must not share pages with unrelated (e.g. torch) host buffers (include/ut.h)."""

    def __init__(self, adj):
        self.n = len(adj)
        ip = np.zeros(self.n + 1, dtype=np.int64)
        for v, a in enumerate(adj):
            ip[v + 1] = ip[v] + len(a)
        ix = np.array([u for a in adj for u in a] or [0], dtype=np.int32)
        self.m = int(ip[-1])
        self._b = [workloads.HostBuffer(ip.nbytes), workloads.HostBuffer(ix.nbytes)]
        self.indptr = self._b[0].array().view(np.int64)
        self.indptr[:] = ip
        self.indices = self._b[1].array().view(np.int32)
        self.indices[:] = ix


def _both(csr_indptr_addr, csr_indices_addr, n, m, seeds, fanouts, seed, g):
    want = oracle.sample(csr_indptr_addr, csr_indices_addr, n, seeds, fanouts, seed)
    got = g.sample(torch.tensor(np.asarray(seeds, dtype=np.int64), device="cuda"), fanouts, seed)
    return want, got.cpu().numpy()


@pytest.mark.parametrize("trial", range(12))
def test_small_random_graphs(trial):
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(2, 400))
    adj = [sorted(set(rng.integers(0, n, size=int(rng.integers(0, 30))).tolist())) for _ in range(n)]
    c = HostCSR(adj)
    with ut.Graph(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m, keep=c) as g:
        for s in range(3):
            seeds = rng.integers(0, n, size=int(rng.integers(1, 20))).tolist()
            fan = [int(x) for x in rng.integers(0, 12, size=int(rng.integers(1, 4)))]
            want, got = _both(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m, seeds, fan,
                              trial * 7 + s, g)
            np.testing.assert_array_equal(got, want)


def test_k5_star_and_tree():
    adj = [[u for u in range(5) if u != v] for v in range(5)]
    c = HostCSR(adj)
    with ut.Graph(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m, keep=c) as g:
        for s in range(10):
            want, got = _both(c.indptr.ctypes.data, c.indices.ctypes.data, 5, c.m, [0], [2], s, g)
            assert len(got) == 3
            np.testing.assert_array_equal(got, want)
    R, D = 300, 23
    adj = [[R + v * D + s for s in range(D)] for v in range(R)] + [[] for _ in range(R * D)]
    c = HostCSR(adj)
    with ut.Graph(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m, keep=c) as g:
        for f in (1, 5, 22, 23, 40):
            want, got = _both(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m,
                              list(range(R)), [f], f, g)
            np.testing.assert_array_equal(got, want)


@pytest.fixture(scope="module")
def products_csr():
    g = workloads.CSRGraph(2_449_029, 61_900_000, seed=3)
    yield g
    g.close()


@pytest.mark.parametrize("opt", ["indptr=host", "indptr=hbm", "indices=hbm"])
def test_products_shaped_minibatches(products_csr, opt):
    c = products_csr
    with ut.Graph(c.indptr_addr, c.indices_addr, c.n_nodes, c.n_edges, keep=c) as g:
        g.set_option(opt)
        rng = np.random.default_rng(1)
        for b in range(3):
            seeds = rng.choice(c.n_nodes, size=1024, replace=False)
            want = oracle.sample(c.indptr_addr, c.indices_addr, c.n_nodes, seeds, [15, 10, 5], b)
            got = g.sample(torch.from_numpy(seeds).cuda(), [15, 10, 5], b).cpu().numpy()
            assert got.size == want.size > 100_000
            np.testing.assert_array_equal(got, want)


def test_fused_sample_then_gather(products_csr):
    c = products_csr
    rows, rb = c.n_nodes, 400
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.addr, rows, rb, 5, threads=0)
    seeds = np.random.default_rng(2).choice(rows, size=1024, replace=False)
    with ut.Graph(c.indptr_addr, c.indices_addr, c.n_nodes, c.n_edges, keep=c) as g, \
            ut.Table(hb.addr, rows, rb) as t:
        nodes = g.sample(torch.from_numpy(seeds).cuda(), [15, 10, 5], 9)
        feats = t[nodes]
        want_nodes = oracle.sample(c.indptr_addr, c.indices_addr, c.n_nodes, seeds, [15, 10, 5], 9)
        want, _ = oracle.gather(hb.addr, rows, rb, want_nodes)
        assert feats.cpu().numpy().tobytes() == want.tobytes()
    hb.close()


def test_errors_and_edge_cases():
    adj = [[1, 2], [0], [0], []]
    c = HostCSR(adj)
    with ut.Graph(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m, keep=c) as g:
        # duplicate seeds collapse; zero fanout keeps the seeds; isolated node
        got = g.sample(torch.tensor([1, 1, 3], device="cuda"), [0], 1).cpu().tolist()
        assert got == [1, 3]
        got = g.sample(torch.tensor([3], device="cuda"), [5, 5], 1).cpu().tolist()
        assert got == [3]
        with pytest.raises(ut.UTError) as e:
            g.sample(torch.tensor([0, 4], device="cuda"), [1], 1)
        assert e.value.code == ut.UT_ERANGE
        # still usable after the error
        got = g.sample(torch.tensor([0], device="cuda"), [2], 1).cpu().tolist()
        assert got == oracle.sample(c.indptr.ctypes.data, c.indices.ctypes.data, 4, [0], [2], 1).tolist()
        small = torch.empty(1, dtype=torch.int64, device="cuda")
        with pytest.raises(ut.UTError):
            ut.ut_sample(g.handle, torch.tensor([0], device="cuda").data_ptr(), 1, [2], 1,
                         small.data_ptr(), 1)
    with pytest.raises(ut.UTError):
        bad = np.array([0, 5, 3], dtype=np.int64)      # indptr[n] != n_edges
        ut.Graph(bad.ctypes.data, c.indices.ctypes.data, 2, 2)


def test_async_sample_gather_dn_and_cuda_graph(products_csr):
    """ut_sample_async + ut_gather_dn: no host sync between sampling and gathering; the whole
    minibatch captured once in a CUDA graph and replayed for new seeds matches the oracle."""
    c = products_csr
    rows, rb = c.n_nodes, 400
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.addr, rows, rb, 6, threads=0)
    fan = [15, 10, 5]
    rng = np.random.default_rng(3)
    with ut.Graph(c.indptr_addr, c.indices_addr, c.n_nodes, c.n_edges, keep=c) as g, \
            ut.Table(hb.addr, rows, rb) as t:
        cap = g.capacity(1024, fan)
        assert cap == min(rows, 1024 * 16 * 11 * 6)
        seeds = torch.empty(1024, dtype=torch.int64, device="cuda")
        nodes = torch.empty(cap, dtype=torch.int64, device="cuda")
        n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        out = torch.empty(cap * rb, dtype=torch.uint8, device="cuda")

        def check(seed_np, salt):
            want_nodes = oracle.sample(c.indptr_addr, c.indices_addr, rows, seed_np, fan, salt)
            n = int(n_dev.item())
            assert n == want_nodes.size
            np.testing.assert_array_equal(nodes[:n].cpu().numpy(), want_nodes)
            want, _ = oracle.gather(hb.addr, rows, rb, want_nodes)
            assert out[: n * rb].cpu().numpy().tobytes() == want.tobytes()

        # eager, asynchronous
        s0 = rng.choice(rows, size=1024, replace=False)
        seeds.copy_(torch.from_numpy(s0))
        g.sample_async(seeds, fan, 21, nodes, n_dev)
        t.gather_dn(nodes, n_dev, out)
        torch.cuda.synchronize()
        check(s0, 21)
        # captured once, replayed with new seeds in the same buffer
        stream = torch.cuda.Stream()
        graph = torch.cuda.CUDAGraph()
        torch.cuda.synchronize()
        with torch.cuda.graph(graph, stream=stream):
            g.sample_async(seeds, fan, 22, nodes, n_dev, stream=stream)
            t.gather_dn(nodes, n_dev, out, stream=stream)
        for _ in range(3):
            s1 = rng.choice(rows, size=1024, replace=False)
            seeds.copy_(torch.from_numpy(s1))
            torch.cuda.synchronize()
            graph.replay()
            torch.cuda.synchronize()
            check(s1, 22)
    hb.close()


def test_gather_dn_counts_on_device():
    rows, rb = 5000, 68
    hb = workloads.HostBuffer(rows * rb, offset=5)
    workloads.fill_table(hb.addr, rows, rb, 8)
    idx = workloads.uniform_idx(3000, rows, 9)
    with ut.Table(hb.addr, rows, rb) as t:
        for n, reorder in [(0, "off"), (1, "off"), (1777, "off"), (3000, "on"), (5000, "on")]:
            t.set_plan(f"reorder={reorder}")
            out = torch.full((3000 * rb,), 0xAB, dtype=torch.uint8, device="cuda")
            t.gather_dn(torch.from_numpy(idx).cuda(), torch.tensor([n], device="cuda"), out)
            m = min(n, 3000)
            want, _ = oracle.gather(hb.addr, rows, rb, idx[:m])
            got = out.cpu().numpy()
            assert got[: m * rb].tobytes() == want.tobytes()
            assert (got[m * rb:] == 0xAB).all()
    hb.close()
