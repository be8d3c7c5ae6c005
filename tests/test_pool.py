"""The library's recycling unified allocator (``ut_pool_*``, csrc/ut_pool.cu; PAPER.md P:530-531,
DESIGN.md R19 / §6e) replayed against oracle/pool_model.py. The bookkeeping runs on the SYSTEM
(malloc) backend without a GPU; the pinned / managed backends, pool tables and their gathers run
under ``-m gpu`` and call through the C ABI."""
import random

import numpy as np
import pytest

import paper_2101_07956_b200 as ut
from oracle.pool_model import PoolError, PoolModel

STAT_KEYS = ("backend_calls", "backend_frees", "recycled_hits", "bytes_live", "bytes_cached",
             "blocks_live", "blocks_cached")


def _ops(seed, n=300, sizes=(0, 1, 300, 512, 700, 1000, 4096, 5000, 65536)):
    rng = random.Random(seed)
    ops, live = [], []
    for _ in range(n):
        r = rng.random()
        if live and r < 0.4:
            ops.append(("free", live.pop(rng.randrange(len(live)))))
        elif r < 0.43:
            ops.append(("release",))
        else:
            ops.append(("alloc", len(ops), rng.choice(sizes)))
            live.append(len(ops) - 1)
    return ops


def replay(pool: "ut.Pool", model: PoolModel, ops):
    """Same operations on both; the library's blocks must map one to one onto the model's ids
    (same reuse decisions), capacities, errors and counters must agree after every step."""
    addr_of, tag_addr, tag_id = {}, {}, {}
    for op in ops:
        if op[0] == "alloc":
            _, tag, size = op
            try:
                mid, mcap = model.allocate(size)
                merr = None
            except PoolError as e:
                merr = e.kind
            if merr:
                with pytest.raises(ut.UTError) as ei:
                    pool.alloc(size)
                assert ei.value.code == ut.UT_ENOMEM
            else:
                addr, cap = pool.alloc(size)
                assert cap == mcap
                if mid == 0:
                    assert addr == 0
                else:
                    # a fresh model id may reuse an address the backend freed earlier
                    if mid in addr_of:
                        assert addr_of[mid] == addr            # recycled: the very block
                    else:                                      # fresh: not a held block
                        held = {addr_of[i] for i in model.live if i != mid} | {
                            addr_of[i] for st in model.cached.values() for i in st}
                        assert addr not in held
                        addr_of[mid] = addr
                tag_addr[tag], tag_id[tag] = addr, mid
        elif op[0] == "free":
            tag = op[1]
            if tag not in tag_id:
                continue
            model.free(tag_id[tag])
            pool.free(tag_addr[tag])
        else:
            model.release_cached()
            pool.release_cached()
        st = pool.stats()
        assert {k: st[k] for k in STAT_KEYS} == model.stats(), op
    for tag in {o[1] for o in ops if o[0] == "alloc"} - {o[1] for o in ops if o[0] == "free"}:
        if tag in tag_id:                                # still live: hand back to both
            model.free(tag_id[tag])
            pool.free(tag_addr[tag])
    st = pool.stats()
    assert {k: st[k] for k in STAT_KEYS} == model.stats() and st["blocks_live"] == 0
    return addr_of


@pytest.mark.parametrize("seed", range(8))
def test_system_pool_matches_model(seed):
    pool, model = ut.Pool("system"), PoolModel()
    replay(pool, model, _ops(seed))
    # recycled blocks are the same addresses: a live block is never handed out twice
    for _ in range(3):
        a, _c = pool.alloc(2000)
        b, _c = pool.alloc(2000)
        assert a != b
        pool.free(a)
        pool.free(b)
        assert pool.alloc(2048)[0] == b                # last freed first (R19)
        pool.free(b)
    pool.close()


@pytest.mark.parametrize("seed", range(4))
def test_system_pool_with_limit_matches_model(seed):
    limit = 3 * 65536
    pool, model = ut.Pool("system", limit_bytes=limit), PoolModel(limit=limit)
    replay(pool, model, _ops(100 + seed, sizes=(512, 4096, 65536, 100000)))
    assert pool.stats()["limit_bytes"] == limit


def test_system_pool_errors_and_sentinel():
    pool = ut.Pool("system")
    assert pool.alloc(0) == (0, 0)
    pool.free(0)                                        # sentinel: no-op
    a, cap = pool.alloc(1000)
    assert cap == 1024 and pool.stats()["backend_calls"] == 1
    pool.free(a)
    with pytest.raises(ut.UTError) as e:                # double free
        pool.free(a)
    assert e.value.code == ut.UT_EINVAL
    x = np.zeros(16, np.uint8)
    with pytest.raises(ut.UTError):                      # foreign pointer
        pool.free(x.ctypes.data)
    b, _ = pool.alloc(600)
    assert b == a
    with pytest.raises(ut.UTError) as e:                 # destroy refuses while a block is live
        pool.close()
    assert e.value.code == ut.UT_EINVAL and "live" in ut.last_error()[1]
    pool.free(b)
    pool.close()
    assert ut._lib.ut_pool_destroy(None) == ut.UT_OK


def test_system_pool_memory_is_usable_and_kept():
    pool = ut.Pool("system")
    a, cap = pool.alloc(5000)
    buf = np.ctypeslib.as_array((np.ctypeslib.ctypes.c_uint8 * cap).from_address(a))
    buf[:] = np.arange(cap) % 251
    pool.free(a)
    b, _ = pool.alloc(5100)                              # same bucket: the same bytes back
    assert b == a and np.array_equal(buf, np.arange(cap) % 251)
    pool.free(b)
    pool.close()


def test_pool_argument_errors():
    L = ut._lib
    assert L.ut_pool_create(7, 0) is None and ut.last_error()[0] == ut.UT_EINVAL
    assert L.ut_pool_create(ut.UT_ALLOC["vmm"], 0) is None
    assert L.ut_pool_alloc(None, 8, None, None) == ut.UT_EINVAL
    assert L.ut_pool_free(None, None) == ut.UT_EINVAL
    assert L.ut_pool_release_cached(None) == ut.UT_EINVAL
    assert L.ut_pool_get_stats(None, None) == ut.UT_EINVAL
    pool = ut.Pool("system")
    with pytest.raises(ut.UTError) as e:                 # not GPU-mapped: no table over it
        pool.table(4, 64)
    assert e.value.code == ut.UT_EINVAL
    assert L.ut_pool_table(pool.handle, None, 0, 64, None) is None
    pool.close()


def test_concurrent_threads_keep_counters_consistent():
    import threading
    pool = ut.Pool("system")

    def work(seed):
        rng = random.Random(seed)
        held = []
        for _ in range(2000):
            if held and rng.random() < 0.5:
                pool.free(held.pop())
            else:
                held.append(pool.alloc(rng.choice((512, 1024, 4096)))[0])
        for a in held:
            pool.free(a)

    th = [threading.Thread(target=work, args=(s,)) for s in range(8)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    st = pool.stats()
    assert st["blocks_live"] == 0 and st["bytes_live"] == 0
    assert st["blocks_cached"] == st["backend_calls"]
    assert st["recycled_hits"] + st["backend_calls"] > 0
    pool.close()


# ---- GPU: the real backends and pool tables -----------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["pinned", "managed"])
def test_gpu_pool_matches_model(kind):
    import torch
    torch.cuda.init()
    pool, model = ut.Pool(kind), PoolModel()
    replay(pool, model, _ops(7, n=150))
    pool.release_cached()
    pool.close()


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["pinned", "managed"])
def test_gpu_pool_tables_gather_and_recycle(kind):
    """Tables over pool blocks gather bit-exactly (oracle), and releasing one hands its block to
    the next table of the same rounded size without a backend call."""
    import torch
    import oracle
    import workloads
    pool = ut.Pool(kind)
    seen = set()
    for i, (rows, rb) in enumerate([(1000, 400), (1000, 400), (800, 500), (3000, 68), (1000, 400)]):
        tab = np.empty(rows * rb, np.uint8)
        workloads.fill_table(tab, rows, rb, seed=i)
        t = pool.table(rows, rb, src=tab)
        seen.add(t.host_addr)
        idx = workloads.uniform_idx(4099, rows, seed=10 + i)
        idx[7] = rows - 1
        out = t.gather(torch.from_numpy(idx).cuda())
        torch.cuda.synchronize()
        exp, bad = oracle.gather(tab, rows, rb, idx)
        assert bad == -1
        assert np.array_equal(out.cpu().numpy().reshape(-1), exp)
        assert t.info()["alloc_kind"] == ut.UT_ALLOC[kind]
        t.close()
    st = pool.stats()
    # 1000 x 400 and 800 x 500 B are one 512-B bucket (400 384 B); 204 000 B is its own size
    assert st["backend_calls"] == 2 and st["recycled_hits"] == 3 and len(seen) == 2
    assert st["blocks_live"] == 0 and st["blocks_cached"] == 2
    pool.close()


@pytest.mark.gpu
def test_gpu_pool_table_on_second_device_or_skip():
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU")
    import oracle
    import workloads
    pool = ut.Pool("managed")
    tab = np.empty(500 * 256, np.uint8)
    workloads.fill_table(tab, 500, 256, seed=3)
    t = pool.table(500, 256, src=tab)
    idx = workloads.uniform_idx(777, 500, seed=4)
    with torch.cuda.device(1):
        out = t.gather(torch.from_numpy(idx).cuda(1))
        torch.cuda.synchronize(1)
    exp, _ = oracle.gather(tab, 500, 256, idx)
    assert np.array_equal(out.cpu().numpy().reshape(-1), exp)
    t.close()
    pool.close()


@pytest.mark.gpu
def test_gpu_pool_tables_from_threads_share_device_resources():
    """Four host threads create, gather from and release pool tables at once on one device: the
    tables' error words come from one shared slab and their scratch (line sharing, reorder) from
    one shared stream-ordered pool that every release trims. Every gather == oracle, every
    out-of-range id reported to its own table only."""
    import threading

    import torch
    import oracle
    import workloads
    pool = ut.Pool("managed")
    errors = []

    def work(k):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            for it in range(6):
                rows, rb = 20000 + 37 * k, (400, 512, 260)[(k + it) % 3]
                with pool.table(rows, rb) as t:
                    t.set_plan(("share=on", "reorder=on", "auto")[(k + it) % 3])
                    workloads.fill_table(t.host_addr, rows, rb, seed=100 * k + it)
                    idx = workloads.uniform_idx(30000, rows, seed=1000 * k + it)
                    bad_at = 1234 + k if it % 2 else -1
                    if bad_at >= 0:
                        idx[bad_at] = rows + k          # this table's only out-of-range id
                    want, want_bad = oracle.gather(t.host_addr, rows, rb, idx)
                    with torch.cuda.stream(st):
                        out = t.gather(torch.from_numpy(idx).cuda(), stream=st)
                    st.synchronize()
                    assert out.cpu().numpy().reshape(-1).tobytes() == want.tobytes()
                    assert t.error_pos(stream=st) == want_bad == bad_at
        except Exception as e:                           # noqa: BLE001 — reported below
            errors.append(f"thread {k}: {e!r}")

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    st = pool.stats()
    assert st["blocks_live"] == 0 and st["recycled_hits"] > 0
    pool.close()


def test_ten_thousand_events_against_the_naive_allocator():
    """SPEC acceptance criterion 6 (allocator recycling): 10,000 random alloc/free events on
    the library's pool — capacities identical to the no-recycling allocator's, fewer or equal
    backend calls, and the same decisions as the recycling model at every step."""
    from oracle.pool_model import NaiveModel
    ops = _ops(4242, n=10000)
    pool, model, naive = ut.Pool("system"), PoolModel(), NaiveModel()
    replay(pool, model, [o for o in ops if o[0] != "release"])
    caps, ncaps, nid = {}, {}, {}
    for o in ops:
        if o[0] == "alloc":
            nid[o[1]], ncaps[o[1]] = naive.allocate(o[2])
            caps[o[1]] = pool.alloc(o[2])
        elif o[0] == "free":
            naive.free(nid[o[1]])
            pool.free(caps[o[1]][0])
    for tag in set(caps) - {o[1] for o in ops if o[0] == "free"}:
        pool.free(caps[tag][0])
    assert {t: c for t, (_, c) in caps.items()} == ncaps
    assert pool.stats()["backend_calls"] <= naive.backend_calls
    pool.close()


@pytest.mark.gpu
def test_recycled_error_word_starts_clear():
    """A table released with an out-of-range id still recorded (never read by error_pos) hands
    its error word back to the shared slab; the next table that takes the word — here the very
    next one, on a non-blocking stream, gathering right away — reports no error of its own, and
    then exactly its own."""
    import torch
    import oracle
    import workloads
    pool = ut.Pool("pinned")
    rows, rb = 3000, 256
    st = torch.cuda.Stream()                              # non-blocking
    for it in range(50):
        with pool.table(rows, rb) as t:
            workloads.fill_table(t.host_addr, rows, rb, seed=it)
            idx = workloads.uniform_idx(5000, rows, seed=it + 1)
            if it % 2 == 0:
                idx[17] = -5                              # left recorded at release
            with torch.cuda.stream(st):
                out = t.gather(torch.from_numpy(idx).cuda(), stream=st)
            st.synchronize()
            want, bad = oracle.gather(t.host_addr, rows, rb, idx)
            assert out.cpu().numpy().reshape(-1).tobytes() == want.tobytes()
            if it % 2:
                assert t.error_pos(stream=st) == -1 == bad   # the previous table's error is gone
    pool.close()


try:
    from hypothesis import given, settings, strategies as hs
except ImportError:                                      # pragma: no cover
    given = None

if given is not None:
    _op = hs.one_of(hs.tuples(hs.just("alloc"), hs.integers(0, 6000)),
                    hs.tuples(hs.just("free"), hs.integers(0, 50)),
                    hs.tuples(hs.just("release"), hs.just(0)))

    @settings(max_examples=150, deadline=None)
    @given(ops=hs.lists(_op, max_size=60), limit=hs.sampled_from([0, 4096, 10240]))
    def test_system_pool_property(ops, limit):
        """Any alloc / free / release sequence, with or without a byte limit: the library's pool
        takes the model's decisions (same capacities, same reuse, same errors, same counters)."""
        seq, live = [], []
        for kind, v in ops:
            if kind == "alloc":
                seq.append(("alloc", len(seq), v))
                live.append(len(seq) - 1)
            elif kind == "free" and live:
                seq.append(("free", live.pop(v % len(live))))
            elif kind == "release":
                seq.append(("release",))
        pool = ut.Pool("system", limit_bytes=limit)
        replay(pool, PoolModel(limit=limit), seq)
        pool.close()
