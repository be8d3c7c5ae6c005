"""Pins for oracle/pool_model.py (the unified allocator's recycling, PAPER.md P:530-531 under
SPEC.md S:178-235's reading, R19): SPEC's worked examples, closed forms and the
comparison with the no-recycling allocator. CPU only."""
import random
from collections import Counter

import pytest

from oracle.pool_model import NaiveModel, PoolError, PoolModel, round_up


def test_spec_examples():
    p = PoolModel()
    assert p.stats() == dict(backend_calls=0, backend_frees=0, recycled_hits=0, bytes_live=0,
                             bytes_cached=0, blocks_live=0, blocks_cached=0)
    b, cap = p.allocate(1000)
    assert cap == 1024 and p.backend_calls == 1
    z, zcap = p.allocate(0)
    assert (z, zcap) == (0, 0) and p.backend_calls == 1
    p.free(z)
    p.free(b)
    b2, cap2 = p.allocate(900)
    assert b2 == b and cap2 == 1024 and p.backend_calls == 1 and p.recycled_hits == 1
    p.free(b2)
    with pytest.raises(PoolError) as e:
        p.free(b2)
    assert e.value.kind == "invalid"


def test_distinct_sizes_and_same_bucket():
    p = PoolModel()
    for k in range(1, 6):
        p.allocate(512 * k)
    assert p.backend_calls == 5
    q = PoolModel()
    b, _ = q.allocate(4096)
    q.free(b)
    q.allocate(4000)
    assert q.backend_calls == 1


def test_rounding():
    assert [round_up(x) for x in (0, 1, 511, 512, 513, 1024, 1025)] == [0, 512, 512, 512, 1024, 1024, 1536]


def _replay(seed, n_ops=400, sizes=(1, 300, 512, 700, 1000, 4096, 5000, 100000)):
    rng = random.Random(seed)
    ops, live = [], []
    for _ in range(n_ops):
        if live and rng.random() < 0.45:
            ops.append(("free", live.pop(rng.randrange(len(live)))))
        else:
            tag = len(ops)
            ops.append(("alloc", tag, rng.choice(sizes)))
            live.append(tag)
    return ops


@pytest.mark.parametrize("seed", range(12))
def test_closed_form_backend_calls_equal_peak_live(seed):
    """With no limit and whole-block reuse by exact rounded size, the backend creates, per
    capacity, exactly as many blocks as were ever live at once; every other request is a hit."""
    ops = _replay(seed)
    p, nv = PoolModel(), NaiveModel()
    ids, nids, caps, ncaps = {}, {}, {}, {}
    live_now, peak = Counter(), Counter()
    n_alloc = 0
    for op in ops:
        if op[0] == "alloc":
            _, tag, size = op
            ids[tag], caps[tag] = p.allocate(size)
            nids[tag], ncaps[tag] = nv.allocate(size)
            c = -(-size // 512) * 512          # the closed form's own rounding
            live_now[c] += 1
            peak[c] = max(peak[c], live_now[c])
            n_alloc += 1
        else:
            tag = op[1]
            p.free(ids[tag])
            nv.free(nids[tag])
            live_now[caps[tag]] -= 1
    assert caps == ncaps                                   # S:216 capacities identical
    assert p.backend_calls == sum(peak.values()) <= nv.backend_calls
    assert p.recycled_hits == n_alloc - p.backend_calls
    st = p.stats()
    assert st["bytes_live"] == sum(c * k for c, k in live_now.items())
    assert st["bytes_cached"] == sum(c * (peak[c] - live_now[c]) for c in peak)
    assert st["blocks_live"] + st["blocks_cached"] == p.backend_calls   # none InUse and Cached
    assert len(set(ids.values())) == p.backend_calls       # every block id came from one call


def test_lifo_reuse_within_bucket():
    p = PoolModel()
    a, _ = p.allocate(600)
    b, _ = p.allocate(700)
    p.free(a)
    p.free(b)
    assert p.allocate(1000)[0] == b and p.allocate(1024)[0] == a


def test_limit_releases_cache_then_fails():
    p = PoolModel(limit=2048)
    a, _ = p.allocate(1024)
    p.allocate(1024)
    p.free(a)
    with pytest.raises(PoolError) as e:       # 1024 live + 1536 > 2048 even with the cache emptied
        p.allocate(1536)
    assert e.value.kind == "oom"
    st = p.stats()
    assert st["backend_frees"] == 1 and st["bytes_cached"] == 0 and st["bytes_live"] == 1024
    q = PoolModel(limit=2048)
    a, _ = q.allocate(1024)
    q.free(a)
    b, cap = q.allocate(2048)                  # fits after the 1024-B block goes back
    assert cap == 2048 and q.backend_frees == 1 and q.backend_calls == 2 and b != a
    r = PoolModel(limit=2048)
    a, _ = r.allocate(1024)
    r.free(a)
    assert r.allocate(1024)[0] == a and r.backend_frees == 0     # a hit never passes the limit


def test_release_cached():
    p = PoolModel()
    blocks = [p.allocate(s)[0] for s in (512, 512, 2048)]
    for b in blocks[:2]:
        p.free(b)
    p.release_cached()
    st = p.stats()
    assert st["backend_frees"] == 2 and st["bytes_cached"] == 0 and st["bytes_live"] == 2048
    assert p.allocate(512)[0] not in blocks                      # a fresh block
