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


# ---- the launch contract (VERDICT r1, next-round task 2) ----------------------------------------
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _json_line(stdout: str) -> dict:
    lines = [l for l in stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, stdout
    return json.loads(lines[0])


def _check_reductions(line: dict, n: int):
    assert line["n_gpus"] == n and line["dry_run"] is True
    per = line["per_gpu"]
    assert [p["gpu"] for p in per] == list(range(n))
    total = sum(p["bytes"] for p in per)
    slowest = max(p["ms"] for p in per)
    # value = sum over GPUs of bytes / max over GPUs of device time
    assert abs(line["value"] - total / (slowest / 1e3) / 1e9) <= 1e-5 * max(1.0, line["value"])
    assert abs(line["ms_per_step"] - slowest / line["steps"]) < 1e-5


def test_bench_gpus2_plain_launch_runs_two_workers():
    """`python bench.py --gpus 2` alone (no torchrun) drives two GPU workers and prints one line
    with n_gpus = 2 and the sum/max reductions over them."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--config", "tiny", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr
    line = _json_line(p.stdout)
    _check_reductions(line, 2)
    assert line["launcher_ranks"] == 1


def test_bench_gpus2_under_torchrun_gloo():
    """The driver's N > 1 launch (torchrun, one rank per GPU, backend gloo here): both ranks
    rendezvous, rank 0 drives the two GPU workers, exactly one JSON line."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run",
                        "--backend", "gloo", "--config", "tiny", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stderr
    line = _json_line(p.stdout)
    _check_reductions(line, 2)
    assert line["launcher_ranks"] == 2


def test_bench_world_size_mismatch_is_refused():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "4", "--dry-run",
                        "--config", "tiny"], capture_output=True, text=True, timeout=120, cwd=ROOT,
                       env=env)
    assert p.returncode != 0 and "WORLD_SIZE=2" in (p.stderr + p.stdout)


def test_reference_arm_uses_gpu0_lists_of_the_ut_arm():
    """Both arms time the same index lists (same seed, GPU 0's rank slice, same cycling), so
    their config blocks agree."""
    spec = bench.workload_spec("tiny")
    ut_lists = bench.make_index_lists(spec, 0, 2, 4, 2101, 1)
    ref_lists = bench.make_index_lists(spec, 0, 2, 4, 2101, 1)
    assert all(np.array_equal(a, b) for a, b in zip(ut_lists, ref_lists))
    a = bench.config_block(spec, ut_lists, 2, 2101)
    b = bench.config_block(spec, ref_lists, 2, 2101)
    assert a == b and a["seed"] == 2101


def test_reference_arm_line_has_the_contract_keys():
    """`--impl reference` (the oracle on the host cores; no GPU needed) prints one line with the
    keys the driver reads, the reference-arm extras, and the same config as the ut arm."""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--config", "tiny", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert p.returncode == 0, p.stderr
    line = _json_line(p.stdout)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e", "impl"):
        assert k in line, k
    assert line["impl"] == "reference" and line["higher_is_better"] is True
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
    spec = bench.workload_spec("tiny")
    lists = bench.make_index_lists(spec, 0, 1, 6, 2101, 1)
    assert line["config"] == bench.config_block(spec, [lists[(3 + s) % 6] for s in range(3)], 1, 2101)
