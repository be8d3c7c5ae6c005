"""Parity of the CUDA gather (through the C ABI) with the oracle, element by element (bytes).

Bar: bit-exact (the gather is a pure copy, reading R3). Inputs come from
``workloads`` only; expected values only from ``oracle``.
"""
import json
import os
import random

import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
ut = pytest.importorskip("paper_2101_07956_b200")

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SENT = 0xAB


def _gather_check(table, host_addr, rows, rb, idx, out_off=0, plan=None, stream=None):
    """Run ut_gather into a sentinel-filled buffer at byte offset out_off; compare with oracle."""
    idx = np.ascontiguousarray(idx, dtype=np.int64)
    n = idx.size
    want, want_bad = oracle.gather(host_addr, rows, rb, idx)
    if plan is not None:
        table.set_plan(plan)
    buf = torch.full((n * rb + out_off + 64,), SENT, dtype=torch.uint8, device="cuda")
    out = buf[out_off:out_off + n * rb]
    idx_d = torch.from_numpy(idx).cuda()
    table.gather(idx_d, out=out, stream=stream)
    bad = table.error_pos(stream)
    got = buf.cpu().numpy()
    assert got[out_off:out_off + n * rb].tobytes() == want.tobytes(), \
        f"mismatch rb={rb} n={n} off={out_off} plan={table.plan}"
    assert (got[:out_off] == SENT).all() and (got[out_off + n * rb:] == SENT).all(), "wrote outside out"
    assert bad == want_bad
    if plan is not None:
        table.set_plan("auto")


def test_paper_worked_example():
    g = json.load(open(os.path.join(GOLDEN, "paper_fig5_example.json")))
    hb = workloads.HostBuffer(5 * 44)      # page-aligned: registration pins whole pages
    feat = hb.array().view(np.float32).reshape(5, 11)
    feat[:] = np.array([[100 * i + j for j in range(11)] for i in range(5)], dtype=np.float32)
    with ut.Table(feat) as t:
        assert (t.rows, t.row_bytes) == (5, 44)
        out = t[torch.tensor(g["idx"], device="cuda")]
        got = out.cpu().numpy().view(np.float32)
        np.testing.assert_array_equal(got, np.array(g["expected"], dtype=np.float32))
        _gather_check(t, feat.ctypes.data, 5, 44, g["idx"])


@pytest.fixture(scope="module")
def pinned_pool():
    """One pinned 48 MiB host region; tables placed inside it are adopted, not re-registered."""
    pool = torch.empty(48 << 20, dtype=torch.uint8, pin_memory=True)
    yield pool


def test_randomized_instances(pinned_pool):
    """>= 1000 random (row width, table base, rows, n, out offset, plan) instances."""
    rng = random.Random(20210119)
    base_addr = pinned_pool.data_ptr()
    widths = [1, 2, 3, 4, 5, 7, 8, 12, 16, 17, 24, 31, 32, 33, 48, 64, 68, 100, 127, 128, 129,
              132, 256, 260, 400, 500, 511, 512, 513, 516, 1024, 1028, 1172, 1372, 2048, 2052,
              2056, 2064, 2076, 2408, 3200, 4092, 4095, 4096, 5000, 8192, 16384]
    plans = [None, "realign", "realignx", "vec16", "vec16x", "narrow", "bulk", "tma4", "paper_naive", "paper_shift"]
    done = 0
    for it in range(1100):
        rb = rng.choice(widths) if it % 3 else rng.randint(1, 6000)
        rows = rng.randint(1, max(1, min(5000, (40 << 20) // rb)))
        off = rng.randrange(0, 128)
        nbytes = rows * rb
        a = pinned_pool[off:off + nbytes].numpy()
        workloads.fill_table(a, rows, rb, seed=it)
        n = rng.choice([0, 1, 2, 3, 31, 32, 33, rng.randint(0, 700)])
        n = min(n, max(1, (4 << 20) // rb))
        idx = workloads.uniform_idx(n, rows, seed=it + 1)
        if n and rng.random() < 0.3:
            idx[rng.randrange(n)] = rows - 1
        if n and rng.random() < 0.3:
            idx[rng.randrange(n)] = 0
        out_off = rng.choice([0, 0, 0, 1, 4, 8, 12, 15])
        t = ut.Table(base_addr + off, rows, rb)
        try:
            assert t.info()["registered"] == 0          # adopted: already pinned
            if rng.random() < 0.4:
                t.set_plan("reorder=on")                # translation-locality visiting order
            t.set_plan("conc=" + rng.choice(["auto", "dense", "sparse"]))   # launch shape
            t.set_plan("runs=" + rng.choice(["auto", "on", "off"]))          # run merge
            t.set_plan("share=" + rng.choice(["auto", "on", "off"]))         # line sharing
            plan = rng.choice(plans)
            if plan is not None:
                try:
                    t.set_plan(plan)
                except ut.UTError:
                    plan = None
                t.set_plan("auto")
            _gather_check(t, base_addr + off, rows, rb, idx, out_off=out_off, plan=plan)
            done += 1
        finally:
            t.close()
    assert done >= 1000


@pytest.mark.parametrize("rb", [1, 3, 4, 8, 13, 16, 68, 100, 400, 512, 2052, 2408, 4096])
@pytest.mark.parametrize("pad", [0, 1, 7, 9, 15])
def test_guard_page_no_over_read(rb, pad):
    """Table ends exactly at a PROT_NONE page; rows placed so the base is misaligned by the
    residue of -(rows*rb) mod 16. Gathers that include the first and last rows, with every
    admissible plan, must not fault (an over-read kills the process) and must match."""
    rows = 37 + pad
    hb = workloads.HostBuffer(rows * rb, kind="guarded")
    a = hb.array()
    workloads.fill_table(a, rows, rb, seed=rb + pad)
    idx = np.array([rows - 1, 0, rows - 1, rows // 2, 0, rows - 1] * 7, dtype=np.int64)
    with ut.Table(hb.addr, rows, rb) as t:
        assert t.info()["registered"] == 1
        for plan in [None, "realign", "realignx", "vec16", "vec16x", "narrow", "bulk", "tma4", "paper_naive", "paper_shift"]:
            try:
                if plan:
                    t.set_plan(plan)
            except ut.UTError:
                continue
            _gather_check(t, hb.addr, rows, rb, idx, out_off=pad % 16)
            t.set_plan("auto")
    torch.cuda.synchronize()
    del a
    hb.close()


def test_empty_single_last_duplicates_and_out_of_range():
    rb, rows = 68, 1000
    hb = workloads.HostBuffer(rows * rb, offset=3)
    workloads.fill_table(hb.array(), rows, rb, 5)
    with ut.Table(hb.addr, rows, rb) as t:
        # n == 0: no launch, out untouched
        buf = torch.full((16,), SENT, dtype=torch.uint8, device="cuda")
        t.gather(torch.empty(0, dtype=torch.int64, device="cuda"), out=buf)
        assert (buf.cpu() == SENT).all()
        _gather_check(t, hb.addr, rows, rb, [rows - 1])
        _gather_check(t, hb.addr, rows, rb, [3, 3, 3])
        _gather_check(t, hb.addr, rows, rb, [5, rows, 7, -1, 9, 1 << 62, -(1 << 62)])
        _gather_check(t, hb.addr, rows, rb, [-3])
        assert t.error_pos() == -1                    # cleared by the previous read
    hb.close()
    hb = workloads.HostBuffer(8)
    hb.array()[:] = np.arange(8, dtype=np.uint8)
    with ut.Table(hb.array(), 1, 8) as t:
        out = t[torch.zeros(5, dtype=torch.int64, device="cuda")]
        assert (out.cpu().numpy() == np.arange(8)).all()
    hb.close()


@pytest.mark.parametrize("rb", [4, 400, 2408])
def test_other_stream_and_consumer_ordering(rb):
    rows = 20000
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.array(), rows, rb, 8)
    s = torch.cuda.Stream()
    idx = workloads.uniform_idx(50000, rows, 9)
    with ut.Table(hb.addr, rows, rb) as t:
        with torch.cuda.stream(s):
            idx_d = torch.from_numpy(idx).cuda()
            out = t.gather(idx_d)
            ids = out[:, :4].contiguous().view(torch.int32).to(torch.int64)   # consumer on s
        s.synchronize()
        np.testing.assert_array_equal(ids.cpu().numpy().reshape(-1), idx & 0xFFFFFFFF)
        _gather_check(t, hb.addr, rows, rb, idx, stream=s)
    hb.close()


@pytest.mark.parametrize("rb", [4, 68, 400, 2052])
@pytest.mark.parametrize("path", ["zero-copy", "pipeline", "pageable"])
def test_gather_host_end_to_end(rb, path, monkeypatch):
    rows = 300_000 if rb < 1000 else 30_000
    hb = workloads.HostBuffer(rows * rb, offset=rb % 7)
    workloads.fill_table(hb.array(), rows, rb, 10)
    idx = workloads.uniform_idx(123_457, rows, 11)
    idx[5] = rows + 3
    want, bad = oracle.gather(hb.addr, rows, rb, idx)
    if path == "pipeline":
        monkeypatch.setenv("UT_HOST_PIPELINE", "1")
    with ut.Table(hb.addr, rows, rb) as t:
        idx_h = torch.from_numpy(idx).pin_memory()
        if path == "pageable":
            out = torch.full((idx.size, rb), SENT, dtype=torch.uint8)
            t.gather_host(idx_h, out_host=out)
        else:
            out = t.gather_host(idx_h)
        assert out.numpy().tobytes() == want.tobytes()
        assert t.error_pos() == bad == 5
    hb.close()


def test_register_adopt_and_release():
    hb = workloads.HostBuffer(1 << 20)
    t = ut.ut_register(hb.addr, 1024, 1024)
    assert ut.ut_table_get_info(t)["registered"] == 1
    t2 = ut.ut_register(hb.addr + 4096, 16, 1024)     # inside pinned pages: adopted
    assert ut.ut_table_get_info(t2)["registered"] == 0
    ut.ut_release(t2)                                 # leaves the pages pinned
    ut.ut_release(t)
    t = ut.ut_register(hb.addr + 4096, 16, 1024)      # unpinned again: registered afresh
    info = ut.ut_table_get_info(t)
    assert info["registered"] == 1 and info["rows"] == 16 and info["dev_addr"] != 0
    ut.ut_release(t)
    hb.close()


@pytest.mark.parametrize("rb", [4, 68, 400, 512, 2408])
def test_reorder_on_large_table(rb):
    """3-GiB table (beyond the ~1-GiB translation reach): auto reorder on, forced off, forced on
    must all equal the oracle, including duplicate and out-of-range indices."""
    tbytes = 3 << 30
    rows = tbytes // rb
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.array(), rows, rb, 12, threads=0)
    n = max(8192, min(300_000, (64 << 20) // rb))
    idx = workloads.uniform_idx(n, rows, 13)
    idx[::1000] = idx[7]
    idx[17] = -2
    idx[n - 1] = rows
    with ut.Table(hb.addr, rows, rb) as t:
        for mode, conc in [("auto", "auto"), ("off", "dense"), ("on", "sparse"), ("on", "dense")]:
            t.set_plan(f"reorder={mode}")
            t.set_plan(f"conc={conc}")
            _gather_check(t, hb.addr, rows, rb, idx, out_off=0)
            _gather_check(t, hb.addr, rows, rb, idx[: n // 3], out_off=4)
    hb.close()


@pytest.mark.parametrize("kind", ["pinned", "managed", "vmm"])
@pytest.mark.parametrize("rb", [68, 400, 4096])
def test_create_library_owned_table(kind, rb):
    """ut_create: the paper's to("unified") with each allocation kind; src copy and fill paths."""
    rows = 20_000
    src = np.empty(rows * rb, np.uint8)
    workloads.fill_table(src, rows, rb, 31)
    idx = workloads.uniform_idx(30_000, rows, 32)
    idx[3] = rows - 1
    want, _ = oracle.gather(src, rows, rb, idx)
    with ut.Table.create(rows, rb, kind, src=src) as t:
        info = t.info()
        assert info["alloc_kind"] == ut.UT_ALLOC[kind] and info["registered"] == 0
        assert t.array().tobytes() == src.tobytes()
        for plan in ["auto", "reorder=on"]:
            t.set_plan(plan)
            out = t[torch.from_numpy(idx).cuda()]
            assert out.cpu().numpy().tobytes() == want.tobytes()
    with ut.Table.create(rows, rb, kind) as t:       # fill in place, no source copy
        workloads.fill_table(t.host_addr, rows, rb, 31)
        out = t[torch.from_numpy(idx).cuda()]
        assert out.cpu().numpy().tobytes() == want.tobytes()


@pytest.mark.parametrize("rb,off", [(16, 0), (400, 0), (512, 0), (2048, 0), (400, 16)])
def test_run_merge_dense_and_adjacent(rb, off):
    """Run merge (vec16 tables): identity, contiguous ranges, shuffled dense selections,
    duplicates and out-of-range indices, with run merge forced on and off."""
    rows = 6000
    hb = workloads.HostBuffer(rows * rb, offset=off)
    workloads.fill_table(hb.addr, rows, rb, 77)
    rng = np.random.default_rng(rb)
    cases = [np.arange(rows), np.arange(100, 900), rng.permutation(rows)[:3000],
             np.sort(rng.choice(rows, 2500, replace=False)), rng.integers(0, rows, 4000)]
    bad = rng.permutation(rows)[:2000].astype(np.int64)
    bad[[3, 700, 1999]] = [rows, -1, rows + 5]
    cases.append(bad)
    with ut.Table(hb.addr, rows, rb) as t:
        for mode in ["runs=on", "runs=off"]:
            t.set_plan(mode)
            for c in cases:
                _gather_check(t, hb.addr, rows, rb, np.asarray(c, dtype=np.int64))
    hb.close()


@pytest.mark.parametrize("rb,off", [(144, 0), (208, 16), (400, 0), (400, 48), (416, 0), (496, 32),
                                    (512, 16), (272, 112)])
def test_neighbour_line_sharing(rb, off):
    """Line sharing (share=on): selected neighbours whose boundary line is fetched
    once by the predecessor's warp. Identity, contiguous ranges (first and last row included),
    dense shuffled and sorted selections, duplicates (several occurrences of a row and of its
    neighbour), out-of-range indices, and the device-side-count form; forced on and off."""
    rows = 6000
    hb = workloads.HostBuffer(rows * rb, offset=off)
    workloads.fill_table(hb.addr, rows, rb, 78)
    rng = np.random.default_rng(rb + off)
    dup = np.repeat(np.arange(200, 400), 3)
    rng.shuffle(dup)
    cases = [np.arange(rows), np.arange(rows)[::-1], np.arange(0, 900), np.arange(rows - 700, rows),
             rng.permutation(rows)[:3000], np.sort(rng.choice(rows, 2500, replace=False)),
             rng.integers(0, rows, 4000), dup, np.array([5]), np.array([rows - 1, rows - 2])]
    bad = rng.permutation(rows)[:2000].astype(np.int64)
    bad[[3, 700, 1999]] = [rows, -1, rows + 5]
    bad[[10, 11]] = [bad[12] - 1 if bad[12] > 0 else 1, rows]   # a neighbour next to a bad index
    cases.append(bad)
    with ut.Table(hb.addr, rows, rb) as t:
        for mode in ["share=on", "share=off"]:
            t.set_plan(mode)
            for c in cases:
                _gather_check(t, hb.addr, rows, rb, np.asarray(c, dtype=np.int64))
        t.set_plan("share=on")
        idx = rng.permutation(rows)[:4000].astype(np.int64)
        want, _ = oracle.gather(hb.addr, rows, rb, idx)
        for k in [0, 1, 2500, 4000]:
            out = torch.full((4000 * rb,), SENT, dtype=torch.uint8, device="cuda")
            n_dev = torch.tensor([k], dtype=torch.int64, device="cuda")
            t.gather_dn(torch.from_numpy(idx).cuda(), n_dev, out)
            got = out.cpu().numpy()
            assert got[:k * rb].tobytes() == want[:k * rb].tobytes()
            assert (got[k * rb:] == SENT).all()
    hb.close()


def test_neighbour_line_sharing_auto_policy():
    """auto takes line sharing for a dense selection of a 400-B table (and never below 128 B or
    for whole-line rows), and the stats show the two launches (slot marking + gather)."""
    rows, rb = 200_000, 400
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.addr, rows, rb, 79)
    idx = np.random.default_rng(1).permutation(rows)[:80_000].astype(np.int64)
    with ut.Table(hb.addr, rows, rb) as t:
        t.stats(reset=True)
        _gather_check(t, hb.addr, rows, rb, idx)
        assert t.stats()["kernel_launches"] == 2
        # the end-to-end form (pinned host output: direct stores) takes it too
        want, _ = oracle.gather(hb.addr, rows, rb, idx)
        t.stats(reset=True)
        got = t.gather_host(torch.from_numpy(idx).pin_memory())
        assert got.numpy().tobytes() == want.tobytes()
        assert t.stats()["share_gathers"] == 1
        t.set_plan("share=off")
        t.stats(reset=True)
        _gather_check(t, hb.addr, rows, rb, idx)
        assert t.stats()["kernel_launches"] == 1
        assert t.stats()["share_gathers"] == 0
    hb.close()


def test_concurrent_gathers_from_threads_and_streams():
    """The header's threading claim: concurrent ut_gather calls on one table from several host
    threads, each on its own stream, are safe and each result is exact."""
    import threading
    rows, rb = 50_000, 400
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.addr, rows, rb, 91)
    lists = [workloads.uniform_idx(20_000 + 997 * k, rows, 100 + k) for k in range(6)]
    wants = [oracle.gather(hb.addr, rows, rb, l)[0] for l in lists]
    errors = []
    with ut.Table(hb.addr, rows, rb) as t:
        def work(k):
            try:
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    idx = torch.from_numpy(lists[k]).cuda()
                    for rep in range(5):
                        if k % 2:
                            t.set_plan("timing=on")
                        out = t.gather(idx, stream=s)
                        s.synchronize()
                        if out.cpu().numpy().tobytes() != wants[k].tobytes():
                            errors.append((k, rep))
            except Exception as e:   # pragma: no cover - reported below
                errors.append((k, repr(e)))
        th = [threading.Thread(target=work, args=(k,)) for k in range(6)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        assert not errors, errors
        st = t.stats()
        assert st["gathers"] >= 30 and st["timed_launches"] <= st["gathers"]
    hb.close()


@pytest.mark.parametrize("rb,base_off,out_off", [(400, 0, 0), (68, 0, 0), (2408, 0, 0), (16, 0, 0),
                                                 (8192, 0, 0), (100, 4, 8), (400, 0, 4), (36, 2, 0)])
@pytest.mark.parametrize("stage", ["on", "off"])
def test_gather_host_staged_tiles(rb, base_off, out_off, stage):
    """ut_gather_host's direct path with and without host-output tile staging (k_staged): tiles
    of consecutive output rows, ragged last tile, out-of-range rows, any admissible alignment
    (stage=on falls back to per-row stores when base/rb/out share no 4-B alignment)."""
    rows = 50_000 if rb < 4096 else 3000
    hb = workloads.HostBuffer(rows * rb, offset=base_off)
    workloads.fill_table(hb.array(), rows, rb, rb)
    n = 12_345
    idx = workloads.uniform_idx(n, rows, rb + 1)
    idx[:3] = [0, rows - 1, 0]
    idx[1000] = -7
    idx[n - 1] = rows
    want, bad = oracle.gather(hb.addr, rows, rb, idx)
    with ut.Table(hb.addr, rows, rb) as t:
        t.set_plan(f"stage={stage}")
        idx_h = torch.from_numpy(idx).pin_memory()
        buf = torch.full((n * rb + out_off + 64,), SENT, dtype=torch.uint8, pin_memory=True)
        out = buf[out_off:out_off + n * rb]
        t.gather_host(idx_h, out_host=out)
        got = buf.numpy()
        assert got[out_off:out_off + n * rb].tobytes() == want.tobytes()
        assert (got[:out_off] == SENT).all() and (got[out_off + n * rb:] == SENT).all()
        assert t.error_pos() == bad == 1000
    hb.close()
