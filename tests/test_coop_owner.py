"""Host-side logic of the cooperative gather (no GPU): the row-block ownership ut_coop_owner
 is a partition of the rows whose per-owner local indices are dense and
injective, with 2-MiB blocks on large tables and >= 64 blocks per rank on small ones."""
import numpy as np
import pytest

ut = pytest.importorskip("paper_2101_07956_b200")


def _owners(rows, rb, world):
    o = np.empty(rows, dtype=np.int64)
    loc = np.empty(rows, dtype=np.int64)
    for i in range(rows):
        o[i], loc[i] = ut.ut_coop_owner(rows, rb, world, i)
    return o, loc


@pytest.mark.parametrize("rows,rb,world", [(1000, 68, 2), (5000, 4, 3), (777, 2408, 4), (64, 1, 8),
                                           (3, 400, 5), (10_000, 512, 1)])
def test_partition_and_dense_local_ids(rows, rb, world):
    o, loc = _owners(rows, rb, world)
    assert ((o >= 0) & (o < world)).all()
    for r in range(world):
        l = loc[o == r]
        assert np.unique(l).size == l.size                 # injective per owner
        if l.size:
            # the owner's tag table has ceil(blocks / world) * R entries (ut_coop_create)
            R = max(1, rows // (64 * world)) if (rows + (2 << 20) // rb - 1) // max(1, (2 << 20) // rb) < 64 * world \
                else max(1, (2 << 20) // rb)
            blocks = (rows + R - 1) // R
            assert l.max() < ((blocks + world - 1) // world) * R


def test_block_size_rule():
    # products-shaped: 2,449,029 x 400 B = 468 blocks of 2 MiB -> fewer than 64*8 -> shrunk
    rows, rb = 2_449_029, 400
    R1 = (2 << 20) // rb
    assert ut.ut_coop_owner(rows, rb, 1, R1 - 1)[0] == 0
    # world 1: one owner, local index = id
    for i in (0, 17, rows - 1):
        assert ut.ut_coop_owner(rows, rb, 1, i) == (0, i)
    # papers-shaped: 111M x 512 B, 2-MiB blocks of 4096 rows, round robin over 8 ranks
    rows, rb = 111_000_000, 512
    assert [ut.ut_coop_owner(rows, rb, 8, b * 4096)[0] for b in range(10)] == [b % 8 for b in range(10)]
    assert ut.ut_coop_owner(rows, rb, 8, 9 * 4096 + 5) == (1, 4096 + 5)
    # products at world 8: R = rows // 512 -> consecutive rows share an owner
    rows, rb = 2_449_029, 400
    R = rows // 512
    assert ut.ut_coop_owner(rows, rb, 8, R - 1)[0] == 0 and ut.ut_coop_owner(rows, rb, 8, R)[0] == 1


def test_invalid_arguments():
    bad = 2**32 - 1
    assert ut.ut_coop_owner(0, 4, 2, 0)[0] == bad
    assert ut.ut_coop_owner(10, 0, 2, 0)[0] == bad
    assert ut.ut_coop_owner(10, 4, 0, 0)[0] == bad
    assert ut.ut_coop_owner(10, 4, 2, -1)[0] == bad
    assert ut.ut_coop_owner(10, 4, 2, 10)[0] == bad


def test_create_rejects_null_table_without_cuda():
    with pytest.raises(ut.UTError):
        ut.ut_coop_create(0, 1, 0, 10)


@pytest.mark.parametrize("rows,rb,world", [(1000, 68, 2), (5000, 4, 3), (777, 2408, 4), (3, 400, 5),
                                           (10_000, 512, 1), (2_449_029, 400, 8)])
def test_partition_ids_invert_ownership(rows, rb, world):
    """The partitions of all ranks hold every row exactly once, and local row l of rank r's
    partition is the row whose ut_coop_owner is (r, l) — the layout the partitioned fetch reads."""
    seen = np.zeros(rows, dtype=np.int64)
    for r in range(world):
        ids = ut.ut_coop_partition_ids(rows, rb, world, r)
        real = ids >= 0
        seen[ids[real]] += 1
        for l in np.flatnonzero(real)[:: max(1, real.sum() // 200)]:     # sampled on big tables
            assert ut.ut_coop_owner(rows, rb, world, int(ids[l])) == (r, int(l))
    assert (seen == 1).all()
    assert ut.ut_coop_partition_ids(rows, rb, world, world).size == 0     # bad rank
