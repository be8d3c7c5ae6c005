"""Pins of the oracle (oracle/ut_oracle.c) against things other than itself.

Each pin is chosen so that a plausible slip in the loop (source stride i*rb instead of
idx*rb, a dropped row, an off-by-one width, a wrong bound check) fails at least one:
  * the paper's worked example (tests/golden/paper_fig5_example.json);
  * brute force over every index vector of length 0..3 on a 4-row table against numpy fancy
    indexing, for many row widths and base offsets (SURVEY.md §8c "Core semantics");
  * special cases that reduce to a library routine: identity -> the table itself,
    a contiguous range -> one slice (memcpy), torch.index_select on a uint8 view;
  * invariants: permutation round trip, duplicate rows, split/concat;
  * self-identifying content decodes to the requested row ids;
  * out-of-range / negative indices -> zero row + first offending position (reading R4),
    n == 0 -> empty.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _table(rows, rb, seed=3, offset=0):
    buf = np.zeros(rows * rb + offset + 16, dtype=np.uint8)
    t = buf[offset:offset + rows * rb]
    workloads.fill_table(t, rows, rb, seed)
    return t


def test_paper_worked_example():
    g = json.load(open(os.path.join(GOLDEN, "paper_fig5_example.json")))
    n, f = g["rows"], g["features"]
    feat = np.array([[100 * i + j for j in range(f)] for i in range(n)], dtype=np.float32)
    out, bad = oracle.gather(feat.view(np.uint8).reshape(-1), n, f * 4, g["idx"])
    assert bad == -1
    got = out.view(np.float32).reshape(len(g["idx"]), f)
    np.testing.assert_array_equal(got, np.array(g["expected"], dtype=np.float32))


@pytest.mark.parametrize("rb", [1, 2, 3, 4, 5, 6, 7, 8, 9, 16, 17, 68, 128, 129])
@pytest.mark.parametrize("offset", [0, 1, 4, 8, 15])
def test_bruteforce_all_short_index_vectors(rb, offset):
    rows = 4
    t = _table(rows, rb, seed=rb * 31 + offset, offset=offset)
    ref = t.reshape(rows, rb)
    count = 0
    for n in range(4):
        for idx in itertools.product(range(rows), repeat=n):
            idx = np.array(idx, dtype=np.int64)
            out, bad = oracle.gather(t, rows, rb, idx)
            assert bad == -1
            assert out.nbytes == n * rb
            np.testing.assert_array_equal(out.reshape(n, rb), ref[idx])
            count += 1
    assert count == 85


@pytest.mark.parametrize("rb", [1, 4, 68, 400, 2052])
def test_identity_is_table(rb):
    rows = 257
    t = _table(rows, rb)
    out, bad = oracle.gather(t, rows, rb, np.arange(rows))
    assert bad == -1
    assert out.tobytes() == t.tobytes()


@pytest.mark.parametrize("rb", [3, 68, 512])
def test_contiguous_range_is_one_slice(rb):
    rows = 1000
    t = _table(rows, rb)
    a, b = 123, 777
    out, _ = oracle.gather(t, rows, rb, np.arange(a, b))
    assert out.tobytes() == t[a * rb:b * rb].tobytes()


def test_matches_torch_index_select():
    torch = pytest.importorskip("torch")
    rows, rb = 5000, 2408
    t = _table(rows, rb, seed=9)
    idx = workloads.uniform_idx(3000, rows, seed=11)
    out, _ = oracle.gather(t, rows, rb, idx)
    ref = torch.index_select(torch.from_numpy(t.reshape(rows, rb)), 0, torch.from_numpy(idx))
    assert out.tobytes() == ref.numpy().tobytes()


def test_self_identifying_rows_decode():
    rows, rb = 100_000, 68
    t = _table(rows, rb, seed=5)
    idx = workloads.uniform_idx(20_000, rows, seed=6)
    out, _ = oracle.gather(t, rows, rb, idx)
    np.testing.assert_array_equal(workloads.decode_row_ids(out, rb), idx)


def test_permutation_round_trip_and_duplicates():
    rows, rb = 1000, 17
    t = _table(rows, rb)
    p = np.random.default_rng(0).permutation(rows).astype(np.int64)
    once, _ = oracle.gather(t, rows, rb, p)
    back, _ = oracle.gather(once, rows, rb, np.argsort(p))
    assert back.tobytes() == t.tobytes()
    out, _ = oracle.gather(t, rows, rb, [3, 3, 3])
    r = out.reshape(3, rb)
    assert (r[0] == r[1]).all() and (r[1] == r[2]).all()
    assert r[0].tobytes() == t[3 * rb:4 * rb].tobytes()


def test_split_concat():
    rows, rb = 4096, 100
    t = _table(rows, rb)
    idx = workloads.uniform_idx(5000, rows, seed=2)
    whole, _ = oracle.gather(t, rows, rb, idx)
    a, _ = oracle.gather(t, rows, rb, idx[:1234])
    b, _ = oracle.gather(t, rows, rb, idx[1234:])
    assert whole.tobytes() == a.tobytes() + b.tobytes()


def test_out_of_range_zero_row_and_first_position():
    rows, rb = 10, 12
    t = _table(rows, rb)
    idx = np.array([1, 10, 2, -1, 9, 1 << 40], dtype=np.int64)
    out, bad = oracle.gather(t, rows, rb, idx)
    assert bad == 1
    r = out.reshape(-1, rb)
    assert not r[1].any() and not r[3].any() and not r[5].any()
    assert r[0].tobytes() == t[rb:2 * rb].tobytes()
    assert r[4].tobytes() == t[9 * rb:10 * rb].tobytes()
    _, bad = oracle.gather(t, rows, rb, [-5])
    assert bad == 0


def test_empty_and_single_row_and_last_row():
    rows, rb = 1, 7
    t = _table(rows, rb)
    out, bad = oracle.gather(t, rows, rb, [])
    assert out.size == 0 and bad == -1
    out, bad = oracle.gather(t, rows, rb, [0, 0])
    assert out.tobytes() == t.tobytes() * 2 and bad == -1
    rows = 99
    t = _table(rows, rb)
    out, _ = oracle.gather(t, rows, rb, [rows - 1])
    assert out.tobytes() == t[(rows - 1) * rb:].tobytes()


def test_raw_address_entry_on_guarded_buffer():
    rows, rb = 333, 13
    hb = workloads.HostBuffer(rows * rb, kind="guarded")
    a = hb.array()
    workloads.fill_table(a, rows, rb, 4)
    out, bad = oracle.gather(hb.addr, rows, rb, [rows - 1, 0])
    assert bad == -1
    assert out[:rb].tobytes() == a[-rb:].tobytes()
    del a
    hb.close()
