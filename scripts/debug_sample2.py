import sys, os, traceback
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
import oracle
import paper_2101_07956_b200 as ut
from test_sample_gpu import HostCSR
for trial in range(12):
    rng = np.random.default_rng(100 + trial)
    n = int(rng.integers(2, 400))
    adj = [sorted(set(rng.integers(0, n, size=int(rng.integers(0, 30))).tolist())) for _ in range(n)]
    c = HostCSR(adj)
    print("trial", trial, "indptr", hex(c.indptr.ctypes.data), "indices", hex(c.indices.ctypes.data), c.indptr.nbytes, c.indices.nbytes, flush=True)
    with ut.Graph(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, c.m, keep=c) as g:
        for s in range(3):
            seeds = rng.integers(0, n, size=int(rng.integers(1, 20))).tolist()
            fan = [int(x) for x in rng.integers(0, 12, size=int(rng.integers(1, 4)))]
            want = oracle.sample(c.indptr.ctypes.data, c.indices.ctypes.data, c.n, seeds, fan, trial * 7 + s)
            st = torch.tensor(np.asarray(seeds, dtype=np.int64), device="cuda")
            try:
                got = g.sample(st, fan, trial * 7 + s)
                print("  n", got.numel(), "want", len(want), flush=True)
                ok = np.array_equal(got.cpu().numpy(), want)
                print("  ok", ok, flush=True)
            except Exception as e:
                print("  EXC", repr(e)[:300], flush=True)
                raise
