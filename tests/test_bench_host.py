"""bench.py host-side helpers (no GPU): workload specs, traffic model, index-list slicing."""
import numpy as np

import bench


def test_traffic_model_matches_direct_count():
    spec = {"row_bytes": 400}
    l = np.array([0, 1, 7, 1000], dtype=np.int64)
    m = bench.traffic_model(spec, [l])
    sect = sum((s + 399) // 32 - s // 32 + 1 for s in (l * 400).tolist())
    lines = sum((s + 399) // 128 - s // 128 + 1 for s in (l * 400).tolist())
    assert m["line_requests_per_step"] == lines
    assert abs(m["sector_floor_mb_per_step"] - sect * 32 / 1e6) < 0.01


def test_workload_specs_match_baseline_configs():
    p = bench.workload_spec("products")
    assert (p["rows"], p["row_bytes"], p["batch"], p["fanouts"]) == (2_449_029, 400, 1024, [15, 10, 5])
    r = bench.workload_spec("reddit")
    assert (r["rows"], r["row_bytes"], r["batch"], r["fanouts"]) == (232_965, 2408, 1000, [25, 10])
    q = bench.workload_spec("papers")
    assert (q["rows"], q["row_bytes"]) == (111_000_000, 512)
    t = bench.workload_spec("tiny")
    assert (t["rows"], t["row_bytes"], t["n"]) == (1024, 68, 512)
    s = bench.workload_spec("sweep:4")
    assert s["rows"] == 1 << 32 and s["n"] == 1 << 20


def test_uniform_lists_differ_per_rank_and_batch():
    spec = bench.workload_spec("tiny")
    a = bench.make_index_lists(spec, 0, 2, 2, 5, 1)
    b = bench.make_index_lists(spec, 1, 2, 2, 5, 1)
    assert not np.array_equal(a[0], a[1]) and not np.array_equal(a[0], b[0])
    assert all(x.dtype == np.int64 and x.max() < 1024 for x in a + b)
