"""N > 1 host logic of bench.py on CPU: world-size-2 gloo process group on 127.0.0.1.

Covers what the multi-GPU run does besides the (per-rank, collective-free) gather: the shared
/dev/shm table created and filled by rank 0 and mapped by every rank, per-rank minibatch
slicing (disjoint roots), and the max-over-ranks timing reduction."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as tmp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, tag, q):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import bench
    import oracle
    import workloads
    try:
        dist = bench.Dist()
        dist.init("gloo")
        spec = {"workload": "t", "kind": "uniform", "config": "t", "rows": 50_000,
                "row_bytes": 36, "n": 4096}
        hb = bench.open_table(spec, rank, world, 77, dist, tag)
        arr = hb.array()
        ids = workloads.decode_row_ids(arr[: 1000 * 36], 36)
        digest = int(np.frombuffer(arr[::997].tobytes(), dtype=np.uint8).astype(np.int64).sum())
        # the per-rank gather (oracle here: no GPU) reads the shared mapping
        lists = bench.make_index_lists(spec, rank, world, 2, 5, 1)
        out, bad = oracle.gather(hb.addr, spec["rows"], 36, lists[0])
        ok_rows = bool((workloads.decode_row_ids(out, 36) == lists[0]).all()) and bad == -1
        gs = bench.workload_spec("products")
        roots = [set(bench.graphsage.sampler_for("products", seed=5).roots(b, rank, world))
                 for b in range(2)]
        value, mx, mw, launches = bench.box_throughput(dist, (rank + 1) * 1_000_000_000,
                                                       (rank + 1) * 100.0, 0.5 + rank, 3)
        q.put((rank, ids[:5].tolist(), digest, ok_rows, [sorted(r)[:3] for r in roots],
               [len(r) for r in roots], value, mx, mw, launches, lists[0][:4].tolist(),
               gs["rows"]))
        dist.barrier()
        hb.close(unlink=(rank == 0))
        dist.close()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, "error", repr(e)))


@pytest.mark.timeout(300)
def test_two_rank_gloo_shared_table_and_reductions():
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    tag = f"pytest_{os.getpid()}"
    procs = [ctx.Process(target=_worker, args=(r, 2, port, tag, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r = q.get(timeout=240)
        assert r[1] != "error", r
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    r0, r1 = res[0], res[1]
    assert r0[1] == r1[1] == [0, 1, 2, 3, 4]          # both ranks see rank 0's fill
    assert r0[2] == r1[2]                              # identical shared bytes
    assert r0[3] and r1[3]                             # rows gathered from the shared mapping
    assert r0[10] != r1[10]                            # per-rank index streams differ
    # disjoint roots per (batch, rank): rank r takes the r-th slice of the root permutation
    assert all(x == 1024 for x in r0[5] + r1[5])
    assert bench_roots(0) and bench_roots(1)
    # max over ranks of device time, sum of bytes: (1e9 + 2e9) / 0.2 s = 15 GB/s
    for r in (r0, r1):
        assert abs(r[6] - 15.0) < 1e-9 and r[7] == 200.0 and r[8] == 1.5 and r[9] == 6
    assert not os.path.exists(f"/dev/shm/ut_bench_{tag}")


def bench_roots(batch):
    from workloads import graphsage
    s = graphsage.sampler_for("products", seed=5)
    a = set(s.roots(batch, 0, 2))
    b = set(s.roots(batch, 1, 2))
    return not (a & b)
