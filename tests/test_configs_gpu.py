"""Full-size parity: every BASELINE.json config, in the launch configuration bench.py times
(auto plan, reorder and launch shape as chosen at that size), compared with the oracle byte for
byte on whole minibatches; plus the traffic model and the JSON contract of bench.py's helpers."""
import numpy as np
import pytest

import oracle
import workloads

torch = pytest.importorskip("torch")
ut = pytest.importorskip("paper_2101_07956_b200")
bench = pytest.importorskip("bench")

pytestmark = pytest.mark.gpu


def _check_lists(spec, lists, extra_plans=()):
    rows, rb = spec["rows"], spec["row_bytes"]
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.addr, rows, rb, 2101, threads=0)
    try:
        with ut.Table(hb.addr, rows, rb) as t:
            for plan in ("auto",) + tuple(extra_plans):
                t.set_plan(plan)
                for l in lists:
                    idx_d = torch.from_numpy(l).cuda()
                    out = t.gather(idx_d)
                    want, bad = oracle.gather(hb.addr, rows, rb, l)
                    got = out.cpu().numpy().reshape(-1)
                    assert got.tobytes() == want.tobytes(), f"{spec['workload']} plan={t.plan}"
                    assert t.error_pos() == bad == -1
            st = t.stats()
            assert st["gathers"] >= len(lists)
    finally:
        hb.close()


@pytest.mark.parametrize("config", ["tiny", "reddit", "products", "papers"])
def test_paper_shaped_configs_full_minibatches(config):
    spec = bench.workload_spec(config)
    lists = bench.make_index_lists(spec, 0, 1, 2, 2101 + 17, 1)
    # rank 1 of 2 as well: the sharded path is the same gather on another root slice
    lists += bench.make_index_lists(spec, 1, 2, 1, 2101 + 17, 1)
    _check_lists(spec, lists, extra_plans=("conc=dense", "conc=auto") if config == "papers" else ())


@pytest.mark.parametrize("rb", [4, 68, 512, 2052])
def test_sweep_table_16gib(rb):
    spec = bench.workload_spec(f"sweep:{rb}")
    lists = bench.make_index_lists(spec, 0, 1, 1, 7, 1)
    lists[0][:3] = [0, spec["rows"] - 1, spec["rows"] // 2]       # first and last row of 2^32 for 4 B
    _check_lists(spec, lists, extra_plans=("reorder=off",))


@pytest.mark.timeout(900)
@pytest.mark.parametrize("config", ["reddit", "products", "papers"])
def test_paper_shaped_configs_managed_table(config):
    """The bench default's table memory at full size: the paper's managed unified tensor
    (ut_create MANAGED, SetPreferredLocation = CPU, filled in place), the auto plan bench.py
    times (line sharing on products), whole minibatches of GPU 0 and of rank 1 of 2, byte for
    byte against the oracle over the same host bytes."""
    spec = bench.workload_spec(config)
    rows, rb = spec["rows"], spec["row_bytes"]
    lists = bench.make_index_lists(spec, 0, 1, 2, 2101, 1)
    lists += bench.make_index_lists(spec, 1, 2, 1, 2101, 1)
    with ut.Table.create(rows, rb, "managed") as t:
        workloads.fill_table(t.host_addr, rows, rb, 2101, threads=0)
        for l in lists:
            out = t.gather(torch.from_numpy(l).cuda())
            want, bad = oracle.gather(t.host_addr, rows, rb, l)
            assert out.cpu().numpy().reshape(-1).tobytes() == want.tobytes(), f"{config} plan={t.plan}"
            assert t.error_pos() == bad == -1
        if config == "products":
            assert t.stats()["share_gathers"] >= len(lists)
