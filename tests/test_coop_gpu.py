"""Parity of the cooperative multi-rank gather (ut_coop_*)
with the oracle, byte for byte, through the C ABI.

The definition is ut_gather's (out[i] = row idx[i]), so the oracle is the same
plain loop. Besides the bytes, the owners' host fetches are checked against what the protocol
promises: every valid row requested by any rank in a step is fetched from host memory exactly
once (sum of the owners' unique rows == |union of the ranks' valid ids|), computed here with
numpy from the inputs alone.

world = 1 runs in-process; world = 2 and 3 run as separate processes that share this box's one
GPU through CUDA IPC (the pool has one GPU per box): the P2P stores and loads then target IPC
mappings of the same device, the same code path that targets NVLink peers on a multi-GPU box.
"""
import os
import socket

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
ut = pytest.importorskip("paper_2101_07956_b200")

pytestmark = pytest.mark.gpu


def _table(rows, rb, seed=11, offset=0):
    hb = workloads.HostBuffer(rows * rb, offset=offset)
    workloads.fill_table(hb.array(), rows, rb, seed=seed)
    return hb


def _lists(rows, n, steps, rank, world, seed, shared=0.5):
    """Per-step index lists that overlap across ranks: a `shared` fraction drawn from a
    step-wide stream every rank sees, the rest from the rank's own stream, shuffled."""
    out = []
    for s in range(steps):
        k = int(n * shared)
        a = workloads.uniform_idx(k, rows, seed=seed * 1000 + s)
        b = workloads.uniform_idx(n - k, rows, seed=seed * 1000 + s + 7919 * (rank + 1))
        l = np.concatenate([a, b])
        rng = np.random.default_rng(seed + 31 * s + rank)
        rng.shuffle(l)
        out.append(np.ascontiguousarray(l, dtype=np.int64))
    return out


def _check_step(c, hb, rows, rb, idx, offset=0):
    want, want_bad = oracle.gather(hb.addr, rows, rb, idx)
    n = idx.size
    buf = torch.full((n * rb + offset + 32,), 0xAB, dtype=torch.uint8, device="cuda")
    out = buf[offset:offset + n * rb]
    c.gather(torch.from_numpy(idx).cuda(), out=out)
    bad = c.error_pos()
    got = buf.cpu().numpy()
    assert got[offset:offset + n * rb].tobytes() == want.tobytes()
    assert (got[:offset] == 0xAB).all() and (got[offset + n * rb:] == 0xAB).all()
    assert bad == want_bad


@pytest.mark.parametrize("rb,offset", [(400, 0), (68, 0), (2408, 0), (512, 0), (3, 0), (36, 5)])
@pytest.mark.parametrize("sync", ["device", "host"])
def test_world1_parity(rb, offset, sync):
    rows = 20_000 if rb <= 512 else 3000
    hb = _table(rows, rb)
    with ut.Table(hb.addr, rows, rb) as t, ut.Coop(t, 6000, world=1, rank=0, sync=sync) as c:
        steps = _lists(rows, 5000, 3, 0, 1, seed=rb)
        steps.append(np.array([], dtype=np.int64))                       # n = 0
        steps.append(np.array([rows - 1, 0, rows - 1], dtype=np.int64))  # edges + duplicate
        steps.append(np.array([5, -1, rows, 7, 5], dtype=np.int64))      # out of range
        for idx in steps:
            _check_step(c, hb, rows, rb, idx, offset)
        st = c.stats()
        assert st["steps"] == len(steps)
        assert st["requested_rows"] == sum(l.size for l in steps)
        valid = [l[(l >= 0) & (l < rows)] for l in steps]
        assert st["owner_requests"] == sum(v.size for v in valid)
        assert st["unique_rows_fetched"] == sum(np.unique(v).size for v in valid)
    hb.close()


def test_world1_full_products_shape():
    """A products-shaped minibatch (2,449,029 x 400 B table, fanout 15/10/5) in one step."""
    from workloads import graphsage
    spec = graphsage.CONFIGS["products"]
    rows, rb = spec["n_nodes"], spec["row_bytes"]
    hb = _table(rows, rb, seed=3)
    idx = graphsage.sampler_for("products", seed=2).minibatch(0)
    with ut.Table(hb.addr, rows, rb) as t, ut.Coop(t, idx.size, world=1, rank=0) as c:
        _check_step(c, hb, rows, rb, idx)
        assert c.stats()["unique_rows_fetched"] == np.unique(idx).size
    hb.close()


def test_bad_arguments():
    hb = _table(100, 16)
    with ut.Table(hb.addr, 100, 16) as t:
        with pytest.raises(ut.UTError):
            ut.ut_coop_create(t.handle, 0, 0, 10)
        with pytest.raises(ut.UTError):
            ut.ut_coop_create(t.handle, 2, 2, 10)
        with pytest.raises(ut.UTError):
            ut.ut_coop_create(t.handle, 1, 0, 0)
        with ut.Coop(t, 10, world=1, rank=0) as c:
            with pytest.raises(ut.UTError):
                c.gather(torch.zeros(11, dtype=torch.int64, device="cuda"))   # n > max_n
    hb.close()


# ---- several processes sharing the GPU ---------------------------------------------------------
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, cfg, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    try:
        import torch.distributed as dist
        dist.init_process_group("gloo", rank=rank, world_size=world)
        torch.cuda.set_device(0)
        rows, rb, n, steps, sync = cfg["rows"], cfg["rb"], cfg["n"], cfg["steps"], cfg["sync"]
        hb = _table(rows, rb, seed=5)              # every rank its own copy (the oracle's input)
        lists = _lists(rows, n, steps, rank, world, seed=rb + world)
        part_kind = cfg.get("partition")            # the fetch then reads only this rank's rows
        if cfg.get("bad"):
            lists[-1] = lists[-1].copy()
            lists[-1][3] = rows + rank              # out of range at position 3
        if cfg.get("empty_rank") == rank:
            lists[1] = np.array([], dtype=np.int64)
        ok, fetched = True, []
        if part_kind:
            ids = ut.Coop.partition_ids(rows, rb, world, rank)
            t = ut.Table.create(ids.size, rb, part_kind)
            workloads.fill_rows(t.host_addr, ids, rb, seed=5)
            c = ut.Coop(t, n, sync=sync, rows=rows)
        else:
            t = ut.Table(hb.addr, rows, rb)
            c = ut.Coop(t, n, sync=sync)
        with t, c:
            prev = 0
            for k, l in enumerate(lists):
                if cfg.get("overflow_rank") == rank and k == 1:
                    # n > max_n on one rank: it errors, but still takes part in the step with no
                    # rows, so the other ranks' device waits complete
                    try:
                        c.gather(torch.zeros(n + 1, dtype=torch.int64, device="cuda"))
                        ok = False
                    except ut.UTError:
                        pass
                    lists[k] = np.array([], dtype=np.int64)
                else:
                    want, want_bad = oracle.gather(hb.addr, rows, rb, l)
                    out = c.gather(torch.from_numpy(l).cuda())
                    got = out.cpu().numpy().reshape(-1)
                    ok &= got.tobytes() == want.tobytes()
                    ok &= c.error_pos() == want_bad
                u = c.stats()["unique_rows_fetched"]
                fetched.append(u - prev)
                prev = u
            dist.barrier()
        hb.close()
        q.put((rank, bool(ok), fetched, [l.tolist() for l in lists]))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, False, repr(e), None))


def _run_world(world, cfg, timeout=240):
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, ok, fetched, lists = q.get(timeout=timeout)
            res[r] = (ok, fetched, lists)
    finally:
        for p in ps:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r in range(world):
        assert res[r][0], f"rank {r}: {res[r][1]}"
    rows = cfg["rows"]
    for s in range(cfg["steps"]):
        ids = np.concatenate([np.array(res[r][2][s], dtype=np.int64) for r in range(world)])
        ids = ids[(ids >= 0) & (ids < rows)]
        assert sum(res[r][1][s] for r in range(world)) == np.unique(ids).size, f"step {s}"


@pytest.mark.parametrize("sync", ["host", "device"])
@pytest.mark.parametrize("world", [2, 3])
def test_processes_share_gpu(world, sync):
    _run_world(world, {"rows": 50_000, "rb": 400, "n": 20_000, "steps": 4, "sync": sync})


@pytest.mark.parametrize("rb", [68, 2408])
def test_processes_unaligned_rows_and_errors(rb):
    _run_world(2, {"rows": 30_000 if rb < 1000 else 4000, "rb": rb, "n": 3000, "steps": 3,
                   "sync": "device", "bad": True, "empty_rank": 1})


def test_processes_one_rank_bad_arguments_does_not_strand_peers():
    _run_world(3, {"rows": 20_000, "rb": 400, "n": 4000, "steps": 3, "sync": "device",
                   "overflow_rank": 1})


@pytest.mark.parametrize("kind", ["managed", "pinned"])
def test_partitioned_tables(kind):
    """Each process holds only its own rows (ut_coop_create_partitioned), in the paper's managed
    memory or pinned memory; outputs still equal the oracle's gather over the whole table."""
    _run_world(2, {"rows": 40_000, "rb": 400, "n": 8000, "steps": 4, "sync": "device",
                   "partition": kind, "bad": True})
    _run_world(3, {"rows": 9000, "rb": 68, "n": 2000, "steps": 3, "sync": "host",
                   "partition": kind})


def test_world1_partitioned_is_the_table():
    rows, rb = 5000, 100
    hb = _table(rows, rb)
    ids = ut.Coop.partition_ids(rows, rb, 1, 0)
    assert (ids[ids >= 0] == np.arange(rows)).all()
    with ut.Table.create(ids.size, rb, "pinned") as t:
        workloads.fill_rows(t.host_addr, ids, rb, seed=11)
        with ut.Coop(t, 3000, world=1, rank=0, rows=rows) as c:
            for idx in _lists(rows, 3000, 2, 0, 1, seed=4):
                _check_step(c, hb, rows, rb, idx)
    hb.close()


def test_world1_randomized_instances():
    """120 random (row width, base offset, rows, n, duplicates, bad ids, out offset) steps through
    one cooperative handle per table, alternating buffer parities."""
    import random
    rng = random.Random(2101_07956)
    for _ in range(12):
        rb = rng.choice([1, 2, 3, 4, 8, 12, 16, 36, 68, 100, 128, 400, 512, 1372, 2052, 2408, 4096])
        rows = rng.randint(1, 4000)
        off = rng.randint(0, 15)
        hb = _table(rows, rb, seed=rb + rows, offset=off)
        with ut.Table(hb.addr, rows, rb) as t, ut.Coop(t, 3000, world=1, rank=0,
                                                        sync=rng.choice(["device", "host"])) as c:
            for _ in range(10):
                n = rng.choice([0, 1, 2, rng.randint(1, 3000)])
                idx = np.array([rng.randrange(rows) for _ in range(n)], dtype=np.int64)
                if n and rng.random() < 0.3:
                    idx[rng.randrange(n)] = rng.choice([-1, rows, rows + 7, -2**40])
                if n > 3 and rng.random() < 0.3:
                    idx[: n // 2] = idx[0]                      # heavy duplication
                _check_step(c, hb, rows, rb, idx, offset=rng.randint(0, 15))
        hb.close()
