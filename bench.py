#!/usr/bin/env python
"""bench.py — unified-tensor gather throughput on B200 (PyTorch-Direct, arXiv 2101.07956).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config products|reddit|papers|tiny|sweep:RB]
                    [--impl ut|reference]

One "step" is one minibatch gather: ``out = table[idx]`` for that step's GraphSAGE-shaped index
list (Listing 2), every row read by GPU threads straight out of the host-pinned,
device-mapped table. Each rank (one per GPU, torchrun for N > 1) gathers its own minibatches from
one shared host table: data parallel by minibatch, no collective on the path ("scaling": "weak").

Printed (rank 0, one JSON line): whole-box useful GB/s (sum of ranks' bytes / max over ranks of
the summed per-step device time), the kernel's roofline against the host-link ceiling measured in
the same run (pinned cudaMemcpy H2D, best of 10 x 1 GiB), the end-to-end figure through
``ut_gather_host`` (host idx in, host rows out), the oracle on the host cores (cpu_baseline), the
paper's CPU-centric baseline (py_baseline), launch count and clocks.

``--impl reference`` times the oracle (oracle/ut_oracle.c, single-threaded plain C) on the host
cores on the same workload, as the reference arm.
"""
from __future__ import annotations

import argparse
import ctypes
import gc
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402
from workloads import graphsage  # noqa: E402

METRIC = "gather GB/s per GPU and per box vs H2D link roofline, 1/2/4/8 B200"
FLUSH_BYTES = 256 << 20      # > 126 MB L2: written between timed steps


# ---- workload ----------------------------------------------------------------------------------
def workload_spec(config: str) -> dict:
    """Table shape + index-list recipe of a config (BASELINE.json configs)."""
    if config in graphsage.CONFIGS:
        c = graphsage.CONFIGS[config]
        names = {"reddit": "reddit-shaped", "products": "ogbn-products-shaped",
                 "papers": "ogbn-papers100M-shaped"}
        return {"workload": names[config], "kind": "graphsage", "config": config,
                "rows": c["n_nodes"], "row_bytes": c["row_bytes"], "batch": c["batch"],
                "fanouts": list(c["fanouts"]), "edges": c["n_edges"]}
    if config == "tiny":
        return {"workload": "tiny", "kind": "uniform", "config": config, "rows": 1024,
                "row_bytes": 68, "n": 512}
    if config.startswith("sweep:"):
        rb = int(config.split(":")[1])
        return {"workload": f"microbenchmark-sweep rb={rb}", "kind": "uniform", "config": config,
                "rows": (16 << 30) // rb, "row_bytes": rb, "n": 1 << 20}
    raise ValueError(config)


def make_index_lists(spec: dict, rank: int, world: int, count: int, seed: int,
                     procs: int) -> list[np.ndarray]:
    """`count` distinct per-rank index lists (generated on the CPU before any timing)."""
    if spec["kind"] == "uniform":
        return [workloads.uniform_idx(spec["n"], spec["rows"], seed=seed + 1000003 * (b * world + rank))
                for b in range(count)]
    rev = bool(spec.get("reverse_fanouts"))
    edges = spec["edges"] if spec["edges"] != graphsage.CONFIGS[spec["config"]]["n_edges"] else None
    jobs = [(spec["config"], seed, b, rank, world, rev, edges) for b in range(count)]
    if procs > 1 and count > 1:
        with mp.get_context("spawn").Pool(min(procs, count)) as pool:
            return pool.map(graphsage.minibatch_job, jobs)
    return [graphsage.minibatch_job(j) for j in jobs]


def open_table(spec: dict, rank: int, world: int, seed: int, dist, tag: str):
    """The shared host feature table: anonymous memory at N=1, a /dev/shm file at N>1 that rank 0
    creates and fills and every rank maps (one copy on the box)."""
    rows, rb = spec["rows"], spec["row_bytes"]
    nbytes = rows * rb
    threads = os.cpu_count() or 1
    if world == 1:
        hb = workloads.HostBuffer(nbytes)
        hb.numa = workloads.interleave(hb.addr, nbytes)
        workloads.fill_table(hb.addr, rows, rb, seed, threads=threads)
        return hb
    name = f"ut_bench_{tag}"
    if rank == 0:
        hb = workloads.HostBuffer(nbytes, kind="shm", name=name, create=True)
        hb.numa = workloads.interleave(hb.addr, nbytes)    # one copy for every socket's GPUs
        workloads.fill_table(hb.addr, rows, rb, seed, threads=threads)
    dist.barrier()
    if rank != 0:
        hb = workloads.HostBuffer(nbytes, kind="shm", name=name, create=False)
    dist.barrier()
    return hb


# ---- distributed plumbing ----------------------------------------------------------------------
class Dist:
    """Rank facts from the torchrun environment; the process group is created by init()."""

    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local_rank = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend: str = "nccl"):
        if self.world > 1:
            import torch.distributed as td
            if backend == "nccl":
                import torch
                torch.cuda.set_device(self.local_rank % torch.cuda.device_count())
                td.init_process_group(backend="nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
            else:
                import datetime
                # the threads harness keeps ranks > 0 waiting while rank 0 fills and times the
                # box (a 57-GB table fill takes minutes): a generous rendezvous timeout
                td.init_process_group(backend=backend, timeout=datetime.timedelta(hours=2))
            self.pg = td

    def barrier(self):
        if self.pg is not None:
            if self.pg.get_backend() == "nccl":
                import torch
                self.pg.barrier(device_ids=[torch.cuda.current_device()])
            else:
                self.pg.barrier()

    def allreduce(self, values: list[float], op: str) -> list[float]:
        if self.pg is None:
            return list(values)
        import torch
        dev = "cuda" if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor(values, dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op={"max": self.pg.ReduceOp.MAX, "sum": self.pg.ReduceOp.SUM}[op])
        return [float(x) for x in t.cpu()]

    def close(self):
        if self.pg is not None:
            self.pg.destroy_process_group()


def box_throughput(dist, nbytes: int, dev_ms: float, wall_s: float, launches: int):
    """Whole-box GB/s = (sum over ranks of useful bytes) / (max over ranks of device time).
    Returns (GB/s, max device ms, max wall s, total launches)."""
    max_dev_ms, max_wall = dist.allreduce([dev_ms, wall_s], "max")
    box_bytes, total_launches = dist.allreduce([float(nbytes), float(launches)], "sum")
    return box_bytes / (max_dev_ms / 1e3) / 1e9, max_dev_ms, max_wall, int(total_launches)


# ---- measurement helpers -----------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks / throttle reasons, sampled every 50 ms. start() returns only once the
    first sample has arrived, so nvidia-smi's own start-up (driver queries, ~1 s) is over before
    anything is timed; mark() brackets the timed region, and the line reports the samples inside
    it (`samples_timed`) next to all samples from the start of warm-up (`samples`). The median
    and the reasons cover warm-up + timing (the timed region alone is ~0.1 s on the default)."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index if isinstance(gpu_index, int) else ",".join(str(g) for g in gpu_index)
        self.lines: list[tuple[float, str]] = []
        self.proc = None
        self.thread = None
        self.window = [None, None]
        self.first = threading.Event()

    def start(self, wait_s: float = 10.0):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, FileNotFoundError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        self.first.wait(wait_s)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.perf_counter(), line.strip()))
            self.first.set()

    def mark(self, which: int) -> None:
        """0: timed region starts, 1: it ends."""
        self.window[which] = time.perf_counter()

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.06)          # one more sample after the timed region
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, mx, reasons, timed = [], [], set(), 0
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        t0, t1 = self.window
        for ts, l in self.lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            if t0 is not None and t1 is not None and t0 <= ts <= t1 + 0.06:
                timed += 1
            for k, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(k)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "samples_timed": timed,
                "window": "warm-up start to timing end, 50-ms nvidia-smi samples"}


def h2d_ceiling(torch, nbytes: int = 1 << 30, reps: int = 10, stream=None, host=None) -> float:
    """Pinned cudaMemcpy H2D ceiling (GB/s) of the current device: best of `reps` copies of
    `nbytes`, CUDA events on `stream` (default: the current stream)."""
    h = host if host is not None else torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    if host is None:
        h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    st = stream if stream is not None else torch.cuda.current_stream()
    best = 0.0
    with torch.cuda.stream(st):
        for _ in range(reps):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            d.copy_(h[:nbytes], non_blocking=True)
            e1.record(st)
            st.synchronize()
            best = max(best, nbytes / e0.elapsed_time(e1) / 1e6)
    del d
    return best


def h2d_ceiling_by_node(torch, dev: int, nbytes: int = 1 << 30):
    """R_link measured once from the table's NUMA placement (node 0, where the fill
    puts or starts it) and once from the GPU-local node — a pinned 1-GiB source bound to each
    node (mbind before first touch, then cudaHostRegister). None on a one-node box (the same
    figure as h2d_memcpy_gbs)."""
    if workloads.numa_nodes() <= 1:
        return None
    cudart = torch.cuda.cudart()
    gnode = workloads.gpu_numa_node(dev)
    out = {"gpu_node": gnode, "gbs": {}}
    for label, node in (("table_node_0", 0), ("gpu_local", gnode)):
        if node < 0 or (label == "gpu_local" and node == 0):
            continue
        hb = workloads.HostBuffer(nbytes)
        try:
            if not workloads.bind_node(hb.addr, nbytes, node):
                out["gbs"][label] = None
                continue
            hb.array()[:] = 1
            if int(cudart.cudaHostRegister(hb.addr, nbytes, 0)) != 0:
                out["gbs"][label] = None
                continue
            try:
                view = torch.frombuffer((ctypes.c_uint8 * nbytes).from_address(hb.addr), dtype=torch.uint8)
                out["gbs"][label] = round(h2d_ceiling(torch, nbytes, 5, host=view), 3)
            finally:
                cudart.cudaHostUnregister(hb.addr)
        finally:
            hb.close()
    return out


def box_topology(torch, devs: list[int]) -> dict:
    """the host-link facts behind R_link / R_concurrent — each GPU's PCI address,
    NUMA node and PCIe link generation / width (read right after the memcpy ceiling, while the
    link is up to speed), and for N > 1 the nearest common ancestor of every GPU pair (same PCIe
    switch, host bridge, NUMA node or across sockets: which GPUs share an uplink)."""
    try:
        import pynvml as nv
        nv.nvmlInit()
    except Exception as e:  # noqa: BLE001 - context only, never fatal
        return {"error": f"nvml: {type(e).__name__}: {e}"[:200]}
    names = {nv.NVML_TOPOLOGY_INTERNAL: "same board", nv.NVML_TOPOLOGY_SINGLE: "one PCIe switch",
             nv.NVML_TOPOLOGY_MULTIPLE: "several PCIe switches",
             nv.NVML_TOPOLOGY_HOSTBRIDGE: "same host bridge", nv.NVML_TOPOLOGY_NODE: "same NUMA node",
             nv.NVML_TOPOLOGY_SYSTEM: "across sockets"}
    out, handles = {"gpus": []}, {}
    try:
        for d in devs:
            p = torch.cuda.get_device_properties(d)
            bus = f"{p.pci_domain_id:08x}:{p.pci_bus_id:02x}:{p.pci_device_id:02x}.0"
            h = nv.nvmlDeviceGetHandleByPciBusId(bus)
            handles[d] = h
            out["gpus"].append({
                "device": d, "pci": bus[4:], "numa_node": workloads.gpu_numa_node(d),
                "pcie_gen": nv.nvmlDeviceGetCurrPcieLinkGeneration(h),
                "pcie_gen_max": nv.nvmlDeviceGetMaxPcieLinkGeneration(h),
                "pcie_width": nv.nvmlDeviceGetCurrPcieLinkWidth(h),
                "pcie_width_max": nv.nvmlDeviceGetMaxPcieLinkWidth(h)})
            g = out["gpus"][-1]       # context, not the roofline
            gts = {1: 2.5, 2: 5.0, 3: 8.0, 4: 16.0, 5: 32.0, 6: 64.0}.get(g["pcie_gen"])
            enc = 0.8 if g["pcie_gen"] in (1, 2) else (242 / 256 if g["pcie_gen"] == 6 else 128 / 130)
            g["theoretical_gbs_per_direction"] = round(gts * g["pcie_width"] * enc / 8, 2) if gts else None
        if len(devs) > 1:
            out["pairs"] = {f"{a}-{b}": names.get(nv.nvmlDeviceGetTopologyCommonAncestor(handles[a], handles[b]), "?")
                            for i, a in enumerate(devs) for b in devs[i + 1:]}
    except Exception as e:  # noqa: BLE001
        out["error"] = f"{type(e).__name__}: {e}"[:200]
    finally:
        try:
            nv.nvmlShutdown()
        except Exception:  # noqa: BLE001
            pass
    return out


def sm_read_ceiling(torch, ut, nbytes: int = 1 << 30, reps: int = 5) -> float:
    """The SM-issued sysmem read ceiling (GB/s): this library's own kernel gathering 512-B rows
    in order from a 1-GiB pinned buffer (whole 128-B lines, sequential addresses) — the most a
    load-based gather can pull over the link, next to the copy engine's memcpy ceiling."""
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    rows = nbytes // 512
    idx = torch.arange(rows, dtype=torch.int64, device="cuda")
    out = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0.0
    with ut.Table(h.data_ptr(), rows, 512) as t:
        for _ in range(reps + 1):
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            t.gather(idx, out=out)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, nbytes / e0.elapsed_time(e1) / 1e6)
    del h, out, idx
    return best


NCU_TRAFFIC = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "ncu_traffic.json")


def ncu_traffic(workload: str, plan: str, table_memory: str, args) -> dict:
    """roofline.traffic from the committed ncu capture of this workload's timed gathers
    (profiles/ncu_traffic.json, written by scripts/ncu_summary.py --traffic): HBM bytes
    (dram__bytes_read.sum + dram__bytes_write.sum) per gather launch, averaged over the captured
    launches, next to the link-side bytes (sysmem sectors x 32) and the algorithmic bytes (n*rb)
    of the same launches. null when no capture matches the workload and plan."""
    try:
        with open(NCU_TRAFFIC) as f:
            rec = json.load(f).get(workload)
    except (OSError, ValueError):
        rec = None
    if (not rec or rec.get("plan") != plan or rec.get("table_memory", table_memory) != table_memory
            or args.plan or args.sample != "cpu" or args.coop != "off"):
        return {"traffic": None}
    detail = {k: rec[k] for k in ("hbm_bytes_per_launch", "hbm_write_bytes_per_launch",
                                  "sysmem_bytes_per_launch", "sysmem_requests_per_launch",
                                  "pcie_read_bytes_per_launch", "algorithmic_bytes_per_launch",
                                  "launches", "source") if k in rec}
    alg = rec.get("algorithmic_bytes_per_launch")
    if alg and rec.get("pcie_read_bytes_per_launch") and rec.get("sysmem_bytes_per_launch"):
        # link bytes per useful byte, split (calibrated by request_rate_probe):
        # 32-B sector over-fetch, then a fixed per-request cost the PCIe counter adds
        req = rec.get("sysmem_requests_per_launch") or 1
        detail["pcie_read_over_algorithmic"] = round(rec["pcie_read_bytes_per_launch"] / alg, 4)
        detail["sectors_over_algorithmic"] = round(rec["sysmem_bytes_per_launch"] / alg, 4)
        detail["pcie_bytes_per_request_beyond_sectors"] = round(
            (rec["pcie_read_bytes_per_launch"] - rec["sysmem_bytes_per_launch"]) / req, 2)
        detail["payload_bytes_per_request"] = round(alg / req, 1)
    return {"traffic": rec["hbm_bytes_per_launch"], "traffic_detail": detail}


def transferred_ncu(value: float, rec: dict) -> dict:
    """transferred GB/s = sysmem sector bytes / time, cross-checked with the PCIe
    read bytes — this run's useful GB/s scaled by the committed ncu capture's per-launch ratios
    for the same workload, plan and table memory (absent when no capture matches)."""
    d = (rec or {}).get("traffic_detail") or {}
    if not d.get("sectors_over_algorithmic"):
        return {}
    return {"transferred_gbs_ncu_sectors": round(value * d["sectors_over_algorithmic"], 3),
            "pcie_read_gbs_ncu": round(value * d["pcie_read_over_algorithmic"], 3)}


def cpu_oracle_rate(table_addr: int, spec: dict, lists: list[np.ndarray], budget_s: float):
    """The oracle as it stands, on this host, over a bounded sample of the same index lists."""
    import oracle
    rb = spec["row_bytes"]
    out = np.empty(max(l.size for l in lists) * rb, dtype=np.uint8)
    # one core on the table's NUMA node (node 0: where the fill first-touched it, or
    # one of the nodes it is striped over); this thread only, restored afterwards
    old_aff = os.sched_getaffinity(0)
    cpu = (workloads.node_cpus(0) or sorted(old_aff))[0]
    try:
        os.sched_setaffinity(0, {cpu})
    except OSError:
        cpu = None
    try:
        done_bytes, done_lists, t0 = 0, 0, time.perf_counter()
        while True:
            l = lists[done_lists % len(lists)]
            oracle.gather_into(table_addr, spec["rows"], rb, l, out)
            done_bytes += l.size * rb
            done_lists += 1
            el = time.perf_counter() - t0
            if el >= budget_s or done_lists >= 64 * len(lists):
                break
    finally:
        if cpu is not None:
            os.sched_setaffinity(0, old_aff)
    cpu_oracle_rate.pinned_cpu = cpu
    return done_bytes / el / 1e9, done_lists, el


# ---- the arms ------------------------------------------------------------------------------------
def run_reference(args, spec, dist):
    """Reference arm: the oracle on the host cores, K timed steps of one minibatch each, over the
    SAME index lists GPU 0 of the ut arm gathers (same seed, same rank slicing, same cycling), so
    the two lines describe one workload. Under torchrun only rank 0 runs it; the other ranks
    exit without work."""
    if dist.rank != 0:
        return
    import oracle
    seed = args.seed
    count = min(args.warmup + args.steps, args.max_lists)
    lists = make_index_lists(spec, 0, args.gpus, count, seed, os.cpu_count() or 1)
    hb = open_table(spec, 0, 1, seed, None, "ref")
    rb = spec["row_bytes"]
    out = np.empty(max(l.size for l in lists) * rb, dtype=np.uint8)
    for s in range(args.warmup):
        oracle.gather_into(hb.addr, spec["rows"], rb, lists[s % count], out)
    step_ms = []
    nbytes = 0
    timed = [lists[(args.warmup + s) % count] for s in range(args.steps)]
    for l in timed:
        t1 = time.perf_counter()
        oracle.gather_into(hb.addr, spec["rows"], rb, l, out)
        step_ms.append((time.perf_counter() - t1) * 1e3)
        nbytes += l.size * rb
    el = sum(step_ms) / 1e3
    value = nbytes / el / 1e9
    line = {"metric": METRIC, "value": round(value, 4), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(el / args.steps * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "impl": "reference",
            "config": config_block(spec, timed, args.gpus, args.seed),
            "step_ms": step_stats(step_ms),
            "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": 1, "cpu_model": cpu_model(),
                             "kind": "oracle",
                             "sample": f"{args.steps} full minibatches of the workload (GPU 0's "
                                       f"lists of the ut arm), single-threaded plain C"},
            "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    hb.close()


def step_stats(ms: list[float]) -> dict:
    """Per-step device (or host) times: the spread a single mean hides."""
    if not ms:
        return {}
    return {"min": round(min(ms), 4), "median": round(statistics.median(ms), 4),
            "max": round(max(ms), 4), "n": len(ms)}


def traffic_model(spec: dict, lists) -> dict:
    """Honest-bytes accounting per step: unique-row bytes, and the link bytes and
    requests a line-aligned warp kernel cannot go below — the 32-B sectors and 128-B lines the
    rows touch (the table starts page-aligned in bench)."""
    rb = spec["row_bytes"]
    uniq, sect, lines = [], [], []
    for l in lists:
        start = l.astype(np.int64) * rb
        uniq.append(np.unique(l).size * rb)
        sect.append(int(((start + rb - 1) // 32 - start // 32 + 1).sum()) * 32)
        lines.append(int(((start + rb - 1) // 128 - start // 128 + 1).sum()))
    m = lambda v: float(np.mean(v)) if v else 0.0
    return {"unique_row_mb_per_step": round(m(uniq) / 1e6, 2),
            "sector_floor_mb_per_step": round(m(sect) / 1e6, 2),
            "line_requests_per_step": round(m(lines), 1)}


def config_block(spec: dict, lists, world: int, seed: int) -> dict:
    rows_per_step = float(np.mean([l.size for l in lists])) if lists else 0.0
    c = {"workload": spec["workload"], "table_rows": spec["rows"], "row_bytes": spec["row_bytes"],
         "seed": seed, "index_lists": "GPU g of N takes rank-g slices (workloads.graphsage / "
                                      "uniform_idx seeded from `seed`); the reference arm times GPU 0's",
         "table_gb": round(spec["rows"] * spec["row_bytes"] / 1e9, 3),
         "rows_per_step_per_gpu": round(rows_per_step, 1),
         "mb_per_step_per_gpu": round(rows_per_step * spec["row_bytes"] / 1e6, 2),
         "parallelism": f"dp{world} (independent minibatch stream per GPU, one shared host table)",
         "l2": "flushed (256 MiB write) between timed steps, outside the per-step events"}
    c.update(traffic_model(spec, lists[:8]))
    if spec["kind"] == "graphsage":
        c.update({"batch": spec["batch"], "fanouts": spec["fanouts"], "graph_edges": spec["edges"]})
    else:
        c["n_per_step"] = spec["n"]
    return c


class _Owned:
    """Stand-in for HostBuffer when the table's memory belongs to the library (ut_create)."""

    def __init__(self, addr):
        self.addr = addr

    def close(self, unlink=False):
        pass


def run_procs(args, spec, dist):
    """One process per GPU (torchrun ranks; --harness procs): each rank registers the shared
    /dev/shm table or holds its own partition (--coop), and gathers its own minibatches. The
    form for the cooperative gather and GPU sampling; the default is run_box."""
    import torch

    rank, world = dist.rank, dist.world
    seed = args.seed
    count = min(args.warmup + args.steps, args.max_lists)
    procs = max(1, (os.cpu_count() or 1) // world)
    lists = make_index_lists(spec, rank, world, count, seed, procs)   # before CUDA init
    if args.presort:   # experiment only: what a perfectly address-ordered list would give
        lists = [np.sort(l) for l in lists]

    ndev = torch.cuda.device_count()
    torch.cuda.set_device(dist.local_rank % ndev)     # > 1 rank per GPU only with --backend gloo
    # host threads of this rank next to its GPU; no-op on single-node boxes
    gnode = workloads.gpu_numa_node(torch.cuda.current_device())
    if gnode >= 0 and workloads.numa_nodes() > 1 and workloads.node_cpus(gnode):
        os.sched_setaffinity(0, workloads.node_cpus(gnode))
    dist.init(args.backend)
    import paper_2101_07956_b200 as ut

    tag = f"{spec['config'].replace(':', '_')}_{os.environ.get('MASTER_PORT', '0')}"
    t_reg = time.perf_counter()
    if args.alloc == "auto":
        # the paper's own allocation (managed memory + its cudaMemAdvise) is the fastest table
        # memory beyond the ~1-GiB translation reach but is process-private; one
        # shared registered table is the only way for N ranks to hold a single copy
        big = spec["rows"] * spec["row_bytes"] > (1 << 30)
        args.alloc = "managed" if (world == 1 and big) else "register"
    partitioned = args.coop != "off" and args.alloc != "register"
    if args.alloc == "register":
        hb = open_table(spec, rank, world, seed, dist, tag)
        t_reg = time.perf_counter()
        table = ut.Table(hb.addr, spec["rows"], spec["row_bytes"])
    elif partitioned:
        # cooperative gather over per-rank partitions: each rank allocates only
        # the rows it owns, of any kind (the paper's managed memory included), one copy in total
        part_ids = ut.Coop.partition_ids(spec["rows"], spec["row_bytes"], world, rank)
        table = ut.Table.create(part_ids.size, spec["row_bytes"], args.alloc)
        workloads.fill_rows(table.host_addr, part_ids, spec["row_bytes"], seed,
                            threads=max(1, (os.cpu_count() or 1) // world))
        hb = _Owned(table.host_addr)
        args.no_cpu = True         # no rank holds the whole table for the host-side baselines
    else:   # the paper's to("unified"): a library-owned table (N = 1 only)
        assert world == 1, "--alloc other than 'register' is single-process"
        table = ut.Table.create(spec["rows"], spec["row_bytes"], args.alloc)
        workloads.fill_table(table.host_addr, spec["rows"], spec["row_bytes"], seed,
                             threads=os.cpu_count() or 1)
        hb = _Owned(table.host_addr)
    reg_s = time.perf_counter() - t_reg
    if args.plan:
        for p in args.plan.split(","):
            table.set_plan(p)
    rb = spec["row_bytes"]
    stream = torch.cuda.current_stream()
    sampler = None
    if args.sample == "gpu":
        sampler = GpuSampling(spec, rank, world, count, seed, ut, torch, args.graph_indptr,
                              "graph" if args.graph else "async" if args.async_sample else "sync")
        lists = sampler.node_lists_for_accounting()
    coop = None
    if args.coop != "off":
        # cooperative gather: rows sampled by several ranks in a step are
        # fetched from host memory once, by their owner, and exchanged through device memory
        assert sampler is None or sampler.mode == "sync", "--coop with --sample gpu: sync sampling only"
        need = sampler.capacity() if sampler is not None else max(l.size for l in lists)
        coop_max = int(dist.allreduce([float(need)], "max")[0])
        coop = ut.Coop(table, coop_max, rank=rank, world=world, sync=args.coop,
                       rows=spec["rows"] if partitioned else None)
    gather = (lambda l, o, st=None: coop.gather(l, out=o, stream=st)) if coop is not None else \
             (lambda l, o, st=None: table.gather(l, out=o, stream=st))
    if sampler is not None and coop is not None:
        sampler.gather_fn = gather
    idx_dev = [torch.from_numpy(l).to("cuda") for l in lists]
    max_n = max(l.size for l in lists)
    out = torch.empty(max_n * rb, dtype=torch.uint8, device="cuda")
    flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")

    # roofline denominator, measured now, on every rank at once (concurrent ceiling at N > 1)
    dist.barrier()
    link = h2d_ceiling(torch)
    link_sum = dist.allreduce([link], "sum")[0]
    sm_ceiling = sm_read_ceiling(torch, ut)

    # parity (outside timing): the first minibatch against the oracle, byte for byte
    parity, parity_lists = None, 0
    if args.check and sampler is not None:
        parity, parity_lists = sampler.check(hb.addr, table, out), 1
        if not parity:
            raise SystemExit(f"rank {rank}: parity failure (GPU sampling + gather)")
    elif args.check:
        # every distinct index list the run gathers is checked against the oracle
        # (bytes), outside timing — all of them up to 16 GB of rows, else the first four
        import oracle
        total = sum(l.size for l in lists) * rb
        n_check = len(lists) if total <= (16 << 30) else min(4, len(lists))
        want_buf = np.empty(max_n * rb, dtype=np.uint8)
        parity = True
        for k in range(n_check):
            l = lists[k]
            if partitioned:
                # no process holds the whole table: build the sub-table of this list's distinct
                # rows (input generation: the table content of those ids, ascending) and let the
                # oracle gather from it with the ids remapped to sub-table rows
                uniq = np.unique(l)
                sub = np.empty(uniq.size * rb, dtype=np.uint8)
                workloads.fill_rows(sub, uniq, rb, seed)
                bad = oracle.gather_into(sub.ctypes.data, uniq.size, rb,
                                         np.searchsorted(uniq, l).astype(np.int64), want_buf)
            else:
                bad = oracle.gather_into(hb.addr, spec["rows"], rb, l, want_buf)
            gather(idx_dev[k], out[: l.size * rb])
            got = out[: l.size * rb].cpu().numpy()
            ok = bool(got.tobytes() == want_buf[: l.size * rb].tobytes()) and \
                (coop.error_pos() if coop is not None else table.error_pos()) == bad
            if not ok:
                raise SystemExit(f"rank {rank}: parity failure on minibatch {k}")
        parity_lists = n_check

    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    # warm-up
    for s in range(args.warmup):
        if sampler is not None:
            sampler.step(s, table, out)
            continue
        l = idx_dev[s % count]
        gather(l, out[: l.numel() * rb])
    torch.cuda.synchronize()
    if sampler is not None and sampler.mode != "sync":
        sampler.device_rows()          # drop the warm-up counts

    table.set_plan("timing=on")
    warm_stats = table.stats(reset=True)      # warm-up (and CUDA-graph capture) counters
    coop0 = coop.stats() if coop is not None else None
    if sampler is not None:
        sampler.mark()
    evs = []
    nbytes = 0
    dist.barrier()
    torch.cuda.synchronize()
    # NVTX range "timed": ncu's --nvtx --nvtx-include "timed/" profiles exactly these launches
    torch.cuda.nvtx.range_push("timed")
    clocks.mark(0)
    t0 = time.perf_counter()
    if sampler is not None and args.pipeline:
        # sample minibatch k+1 (its own stream) while minibatch k is gathered: the whole loop is
        # one timed region on the gather stream; every step writes > L2 (no flush, stated)
        nbytes, ms = sampler.pipelined(args.warmup, args.steps, table, out)
        e0 = e1 = None
        evs = [ms]
    for s in range(0 if (sampler is not None and args.pipeline) else args.steps):
        flush.zero_()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        if sampler is not None:
            nbytes += sampler.step(args.warmup + s, table, out) * rb
        else:
            l = idx_dev[(args.warmup + s) % count]
            gather(l, out[: l.numel() * rb], stream)
            nbytes += l.numel() * rb
        e1.record(stream)
        evs.append((e0, e1))
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    if sampler is not None and sampler.mode != "sync":
        nbytes += sampler.device_rows() * rb
    dist.barrier()
    wall = time.perf_counter() - t0
    clocks.mark(1)
    clk = clocks.stop()
    st = table.stats(reset=True)
    table.set_plan("timing=off")
    dev_ms = evs[0] if (sampler is not None and args.pipeline) else sum(a.elapsed_time(b) for a, b in evs)

    own_launches = st["kernel_launches"]
    # the gather variant of the timed steps: the table's plan, "+share" when the gathers took
    # neighbour line sharing
    # (a captured CUDA graph replays the gathers without passing through ut_gather: its capture,
    # during warm-up, is where the choice shows)
    shared = st.get("share_gathers") or (args.sample != "cpu" and warm_stats.get("share_gathers"))
    plan_label = table.plan + ("+share" if shared else "")
    coop_block = None
    if coop is not None:
        c1 = coop.stats()
        own_launches += c1["kernel_launches"] - coop0["kernel_launches"]
        req = c1["requested_rows"] - coop0["requested_rows"]
        uniq = c1["unique_rows_fetched"] - coop0["unique_rows_fetched"]
        req_all, uniq_all = dist.allreduce([float(req), float(uniq)], "sum")
        coop_block = {"sync": args.coop, "ranks": world,
                      "requested_rows_per_step_all_ranks": round(req_all / args.steps, 1),
                      "host_rows_per_step_all_ranks": round(uniq_all / args.steps, 1),
                      "host_bytes_fraction": round(uniq_all / max(1.0, req_all), 4),
                      "this_rank_fetch_rows_per_step": round(uniq / args.steps, 1),
                      "block_rows": c1["block_rows"], "region_bytes": c1["region_bytes"],
                      "note": "value counts useful rows (n*rb per rank); the host link moved "
                              "host_bytes_fraction of them; roofline.achieved is host-fetched "
                              "bytes / fetch-kernel time"}
    if sampler is not None:
        own_launches += sampler.timed_launches(args.steps)
    value, max_dev_ms, max_wall, launches = box_throughput(dist, nbytes, dev_ms, wall,
                                                           own_launches)
    per_gpu = nbytes / (dev_ms / 1e3) / 1e9
    kern_ms = st["gather_kernel_ms"] / max(1, st["timed_launches"])
    kern_bytes = nbytes / max(1, st["timed_launches"])
    if coop is not None:    # the gather kernels fetch the owners' unique rows only
        kern_bytes = (c1["unique_rows_fetched"] - coop0["unique_rows_fetched"]) * rb / max(1, st["timed_launches"])
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9 if kern_ms > 0 else None   # None: graph replay

    # end to end: host idx in (pinned), host rows out (pinned), through ut_gather_host
    e2e = None
    if not args.no_e2e and sampler is None and coop is None:
        idx_host = [torch.from_numpy(x).pin_memory() for x in lists]
        out_host = torch.empty(max_n * rb, dtype=torch.uint8, pin_memory=True)
        for s in range(min(2, count)):
            table.gather_host(idx_host[s], out_host=out_host)
        e_sec, e_bytes, h2d, d2h = 0.0, 0, 0, 0
        for s in range(args.steps):
            ih = idx_host[(args.warmup + s) % count]
            flush.zero_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            table.gather_host(ih, out_host=out_host)
            e_sec += time.perf_counter() - t1
            e_bytes += ih.numel() * rb
            h2d += ih.numel() * 8
            d2h += ih.numel() * rb
        mx = dist.allreduce([e_sec], "max")[0]
        e_tot = dist.allreduce([float(e_bytes)], "sum")[0]
        e2e = {"value": round(e_tot / mx / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
               "path": "ut_gather_host: idx H2D copy, then the gather kernel stores rows into pinned host memory"}
        # the paper's own pipeline (Listing 2): CPU-sampled index list -> GPU rows for training;
        # pinned idx H2D, gather into HBM, then an 8-byte read-back of the step's result
        f_sec, f_bytes = 0.0, 0
        probe = torch.empty(1, dtype=torch.int64, pin_memory=True)
        for s in range(args.steps):
            ih = idx_host[(args.warmup + s) % count]
            flush.zero_()
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            idx_d = ih.to("cuda", non_blocking=True)
            res = table.gather(idx_d, out=out[: ih.numel() * rb])
            probe.copy_(res[:8].view(torch.int64), non_blocking=False)
            f_sec += time.perf_counter() - t1
            f_bytes += ih.numel() * rb
            if os.environ.get("UT_BENCH_DEBUG"):
                print(f"to_hbm step {s}: {(time.perf_counter() - t1) * 1e3:.3f} ms, n={ih.numel()}",
                      file=sys.stderr)
        mx = dist.allreduce([f_sec], "max")[0]
        f_tot = dist.allreduce([float(f_bytes)], "sum")[0]
        e2e["to_hbm"] = {"value": round(f_tot / mx / 1e9, 3), "unit": "GB/s",
                         "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": 8,
                         "path": "Table.gather with a pinned host idx: idx H2D, gather into HBM, "
                                 "8-B read-back of the result (the paper's Listing 2 pipeline)"}
        del out_host, idx_host

    # optional NCCL all-reduce smoke step (SURVEY §2.3 ii): off the gather path, untimed
    ar = None
    if args.allreduce_smoke and world > 1:
        g = torch.full((1 << 20,), float(rank + 1), dtype=torch.float32, device="cuda")
        t1 = time.perf_counter()
        dist.pg.all_reduce(g)
        torch.cuda.synchronize()
        ar = {"ok": bool((g == world * (world + 1) / 2).all().item()), "bytes": g.numel() * 4,
              "ms": round((time.perf_counter() - t1) * 1e3, 3), "backend": dist.pg.get_backend()}

    # per-box roofline term: host DRAM read bandwidth over the table (all host cores, rank 0)
    dram = None
    if rank == 0 and not args.no_cpu:
        import baselines
        dram = round(baselines.host_read_gbs(hb.addr, min(spec["rows"] * spec["row_bytes"], 8 << 30)), 2)

    # context baselines on rank 0 at N=1: the oracle and the paper's CPU-centric path
    cpu_base, py_base = None, None
    if rank == 0 and world == 1 and not args.no_cpu:
        v, nl, el = cpu_oracle_rate(hb.addr, spec, lists, args.cpu_budget)
        cpu_base = {"value": round(v, 4), "unit": "GB/s", "cores": 1, "cpu_model": cpu_model(), "kind": "oracle",
                    "sample": f"{nl} minibatches of the workload in {el:.1f} s, single-threaded plain C"}
        py_base = cpu_staged_baseline(torch, hb.addr, spec, lists, args)
        py_base.pop("_raw", None)

    if rank == 0:
        n_launch = int(launches)
        cfg = config_block(spec, [lists[(args.warmup + s) % count] for s in range(args.steps)],
                           world, args.seed)
        sect_ratio = (cfg["sector_floor_mb_per_step"] / cfg["mb_per_step_per_gpu"]
                      if cfg.get("mb_per_step_per_gpu") else None)
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(max_dev_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic (self-identifying fp32-row table, GraphSAGE-shaped index lists)",
            "config": cfg,
            "per_gpu_gbs": round(per_gpu, 3),
            "transferred_gbs_sector_floor": round(value * sect_ratio, 3) if sect_ratio else None,
            # rows < 128 B are bound by the link's request rate, not bytes
            "line_requests_per_s": (round(cfg["line_requests_per_step"] * world / (max_dev_ms / args.steps / 1e3))
                                    if cfg.get("line_requests_per_step") else None),
            "h2d_memcpy_gbs": round(link, 3),
            "h2d_memcpy_concurrent_gbs": round(link_sum, 3),
            "host_dram_read_gbs": dram,
            "box_roofline_gbs": round(min(link_sum, dram), 3) if dram else round(link_sum, 3),
            "frac_of_link": round(per_gpu / link, 4),
            "sm_read_ceiling_gbs": round(sm_ceiling, 3),
            "frac_of_sm_read_ceiling": round(per_gpu / sm_ceiling, 4),
            "plan": plan_label,
            "table_memory": args.alloc + (" (per-rank partitions, ut_coop_create_partitioned)" if partitioned else ""),
            "numa": {"nodes": workloads.numa_nodes(), "gpu_node": gnode,
                     "table_policy": "interleave" if getattr(hb, "numa", 0) > 1 else "single node / default"},
            "roofline": {"bound": "pcie_h2d",
                         "achieved": round(achieved, 3) if achieved is not None else None,
                         "peak": round(link, 3), "unit": "GB/s",
                         "frac": round(achieved / link, 4) if achieved is not None else None,
                         **ncu_traffic(spec["workload"], plan_label, args.alloc, args),
                         "kernel": f"gather {plan_label} (device time of the gather kernel alone, CUDA events on its stream)",
                         "peak_source": "pinned cudaMemcpy H2D measured in this run (best of 10 x 1 GiB)",
                         "sm_read_ceiling": round(sm_ceiling, 3)},
            "cpu_baseline": cpu_base, "py_baseline": py_base, "e2e": e2e,
            "gpu_launches": n_launch, "clocks": clk,
            "sampling": sampler.report(args.steps) if sampler is not None else None,
            "ranks_per_gpu": max(1, world // max(1, torch.cuda.device_count())),
            "parity_checked": parity, "parity_lists_checked": parity_lists,
            "register_s": round(reg_s, 3), "allreduce_smoke": ar,
            "coop": coop_block,
            "wall_ms_per_step": round(max_wall / args.steps * 1e3, 3),
        }
        print(json.dumps(line), flush=True)
    dist.barrier()
    if coop is not None:
        coop.close()
    table.close()
    dist.barrier()
    if world > 1 and rank == 0:
        hb.close(unlink=True)
    else:
        hb.close()


# ---- the default harness: one process, ONE table, one host thread per GPU ----------------------
def run_threads(n: int, fn):
    """fn(g) for g in 0..n-1 on n threads at once; results in GPU order; re-raises a failure."""
    res, errs = [None] * n, [None] * n

    def body(g):
        try:
            res[g] = fn(g)
        except BaseException as e:  # noqa: BLE001 - re-raised below on the main thread
            errs[g] = e

    ts = [threading.Thread(target=body, args=(g,), name=f"gpu{g}") for g in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for e in errs:
        if e is not None:
            raise e
    return res


def mem_available() -> int:
    """Host MemAvailable in bytes (0 when unknown)."""
    try:
        with open("/proc/meminfo") as f:
            for line in f:
                if line.startswith("MemAvailable:"):
                    return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


def box_table(spec: dict, args, ut):
    """The box's host feature table(s), shared by the GPUs of the process. Returns
    (tables, owners, kind): one table, or with --numa replica one per host NUMA node (SURVEY §8e:
    "one replica per socket if RAM allows, so every GPU reads locally"; each GPU then gathers from
    the replica on its own node, `replica_of`).

    auto/managed: the paper's own unified-tensor allocation — cudaMallocManaged with
    SetPreferredLocation = CPU and SetAccessedBy = each GPU (Table 2; ut_create
    extends AccessedBy to a device the first time it gathers). On this pool it is the only host
    memory kind that reads random rows at link speed at any table size (managed 50.7 GB/s for
    random 512-B rows over 53 GB; registered / pinned / VMM host memory 25.7-29, profiles/r2/
    shared_table_probe.jsonl) — and it is process-private, which is why one process drives all
    GPUs. register: an anonymous mmap pinned in place (ut_register); pinned / vmm: ut_create."""
    rows, rb = spec["rows"], spec["row_bytes"]
    kind = "managed" if args.alloc == "auto" else args.alloc
    threads = os.cpu_count() or 1
    if kind == "register":
        hb = workloads.HostBuffer(rows * rb)
        hb.numa = workloads.interleave(hb.addr, rows * rb)
        workloads.fill_table(hb.addr, rows, rb, args.seed, threads=threads)
        import paper_2101_07956_b200 as _ut
        return [_ut.Table(hb.addr, rows, rb)], [hb], kind
    nodes = workloads.numa_nodes()
    if kind == "managed" and args.numa == "replica":
        k = args.numa_replicas or max(nodes, 1)
        avail = mem_available()
        if avail and k * rows * rb > 0.85 * avail:
            note = (f"{k} replicas of {rows * rb / 1e9:.1f} GB do not fit 85 % of MemAvailable "
                    f"({avail / 1e9:.1f} GB): one table instead")
            tables, owners, kind = box_table(spec, argparse.Namespace(**{**vars(args), "numa": "auto"}), ut)
            owners[0].numa = {**owners[0].numa, "replica_request": note}
            return tables, owners, kind
        tables, owners = [], []
        for r in range(k):
            node = r % max(nodes, 1)
            table = ut.Table.create(rows, rb, kind)
            owned = _Owned(table.host_addr)
            try:
                table.numa_place(node)
                how = f"ut_numa_place(node {node})"
            except ut.UTError as e:
                how = f"first touch by node {node}'s CPUs (ut_numa_place: {str(e)[:120]})"
            cpus = workloads.node_cpus(node) or list(range(threads))
            pinned = workloads.fill_table_on(table.host_addr, rows, rb, args.seed, cpus)
            owned.numa = {"replica": r, "node": node, "placement": how,
                          "fill": f"{len(cpus)} threads pinned to node {node}'s CPUs"
                                  + ("" if pinned else " (pinning failed: unpinned threads)")}
            tables.append(table)
            owners.append(owned)
        return tables, owners, kind
    table = ut.Table.create(rows, rb, kind)
    owned = _Owned(table.host_addr)
    # the box's one table NUMA-interleaved (2-MiB stripes placed by SetPreferredLocation
    # = host NUMA node, before the fill first-touches them); a no-op policy on one-node boxes
    if kind == "managed" and (args.numa == "interleave" or (args.numa == "auto" and nodes > 1)):
        t0 = time.perf_counter()
        try:
            table.numa_interleave(max(nodes, 1))
            owned.numa = {"policy": f"interleave over {max(nodes, 1)} node(s), 2-MiB stripes "
                                    "(ut_numa_interleave)", "advise_s": round(time.perf_counter() - t0, 3)}
        except ut.UTError as e:
            owned.numa = {"policy": "first touch by the fill threads (interleave requested, not "
                                    f"available: {str(e)[:160]})"}
    else:
        owned.numa = {"policy": "first touch by the fill threads" + ("" if nodes > 1 else " (one NUMA node)")}
    workloads.fill_table(table.host_addr, rows, rb, args.seed, threads=threads)
    return [table], [owned], kind


def replica_of(g_dev: int, g: int, nrep: int) -> int:
    """The replica GPU g gathers from: the one on its device's NUMA node, else g mod replicas."""
    if nrep <= 1:
        return 0
    node = workloads.gpu_numa_node(g_dev)
    return node if 0 <= node < nrep and workloads.numa_nodes() >= nrep else g % nrep


class BoxWorker:
    """GPU g's share of a box run: its minibatch index lists resident in HBM, its output and
    L2-flush buffers and a stream of its own. Every method runs on the calling thread with
    device g made current (CUDA's current device is per host thread)."""

    def __init__(self, g: int, torch, table, spec: dict, lists, args):
        torch.cuda.set_device(g)
        self.g, self.torch, self.table, self.spec, self.args = g, torch, table, spec, args
        self.rb = spec["row_bytes"]
        self.lists = lists
        self.stream = torch.cuda.Stream()
        self.max_n = max(l.size for l in lists)
        with torch.cuda.stream(self.stream):
            self.idx = [torch.from_numpy(l).to("cuda") for l in lists]
            self.out = torch.empty(self.max_n * self.rb, dtype=torch.uint8, device="cuda")
            self.flush = torch.empty(FLUSH_BYTES, dtype=torch.uint8, device="cuda")
            self.flush.zero_()      # loads torch's fill kernel now, not inside a timed step
        self.stream.synchronize()

    coop = None      # --coop device: this GPU's rank of the in-process cooperative gather
    sampler = None   # --sample gpu: this GPU's sampler (GpuSampling, sync mode)

    def gather(self, k: int) -> int:
        if self.sampler is not None:     # sample this step's minibatch on the GPU, then gather
            with self.torch.cuda.stream(self.stream):
                return self.sampler.step(k, self.table, self.out) * self.rb
        l = self.idx[k % len(self.idx)]
        if self.coop is not None:
            self.coop.gather(l, out=self.out[: l.numel() * self.rb], stream=self.stream)
        else:
            self.table.gather(l, out=self.out[: l.numel() * self.rb], stream=self.stream)
        return l.numel() * self.rb

    def error_pos(self) -> int:
        return (self.coop.error_pos(self.stream) if self.coop is not None
                else self.table.error_pos(self.stream))

    def parity(self, host_addr: int, budget_bytes: int) -> int:
        """Byte-exact check of this GPU's lists against the oracle, outside timing (SURVEY §4
        T2): every list while the rows fit `budget_bytes`, at least two. Returns lists checked."""
        import oracle
        if self.sampler is not None:     # sampled node list and its rows, both against the oracle
            with self.torch.cuda.stream(self.stream):
                if not self.sampler.check(host_addr, self.table, self.out):
                    raise SystemExit(f"GPU {self.g}: parity failure (GPU sampling + gather)")
            return 1
        rb = self.rb
        want = np.empty(self.max_n * rb, dtype=np.uint8)
        checked, total = 0, 0
        for k, l in enumerate(self.lists):
            if checked >= 2 and total + l.size * rb > budget_bytes:
                break
            bad = oracle.gather_into(host_addr, self.spec["rows"], rb, l, want)
            self.gather(k)
            self.stream.synchronize()
            got = self.out[: l.size * rb].cpu().numpy()
            if got.tobytes() != want[: l.size * rb].tobytes() or self.error_pos() != bad:
                raise SystemExit(f"GPU {self.g}: parity failure on minibatch {k}")
            checked += 1
            total += l.size * rb
        return checked

    def warmup(self) -> None:
        for s in range(self.args.warmup):
            self.gather(s)
        self.stream.synchronize()

    def timed(self, start) -> dict:
        """K steps, each bracketed by CUDA events on this GPU's stream, the L2 flushed between
        steps outside the events. `start` (a threading.Barrier) releases every GPU at once."""
        torch, args = self.torch, self.args
        self.stream.synchronize()
        start.wait()
        torch.cuda.nvtx.range_push("timed")    # ncu --nvtx-include "timed/" profiles these
        t0 = time.perf_counter()
        if self.sampler is not None and args.pipeline:
            # sample minibatch k+1 (its own stream) while minibatch k is gathered; one timed
            # region for the K steps (every step writes > L2: no flush, stated in the line)
            nbytes, ms = self.sampler.pipelined(args.warmup, args.steps, self.table, self.out)
            torch.cuda.nvtx.range_pop()
            return {"bytes": nbytes, "ms": [ms], "wall_s": time.perf_counter() - t0}
        evs, nbytes = [], 0
        for s in range(args.steps):
            with torch.cuda.stream(self.stream):
                self.flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(self.stream)
            nbytes += self.gather(args.warmup + s)
            e1.record(self.stream)
            evs.append((e0, e1))
        self.stream.synchronize()
        wall = time.perf_counter() - t0
        torch.cuda.nvtx.range_pop()
        return {"bytes": nbytes, "ms": [a.elapsed_time(b) for a, b in evs], "wall_s": wall}

    def e2e(self, start) -> dict:
        """End to end through the public API, per step: (1) ut_gather_host — pinned host idx in,
        pinned host rows out; (2) the paper's Listing 2 pipeline — pinned idx H2D, gather into
        HBM, an 8-B read-back of the result. Host wall time per step; all GPUs at once."""
        torch, args, rb = self.torch, self.args, self.rb
        idx_host = [torch.from_numpy(x).pin_memory() for x in self.lists]
        out_host = torch.empty(self.max_n * rb, dtype=torch.uint8, pin_memory=True)
        probe = torch.empty(1, dtype=torch.int64, pin_memory=True)
        with torch.cuda.stream(self.stream):
            self.idx_up = torch.empty(self.max_n, dtype=torch.int64, device="cuda")
        # warm-up: the largest list first, so the library's device scratch has its final size
        big = max(range(len(idx_host)), key=lambda k: idx_host[k].numel())
        for k in [big] + list(range(min(2, len(idx_host)))):
            self.table.gather_host(idx_host[k], out_host=out_host, stream=self.stream)
        r = {"e_sec": 0.0, "f_sec": 0.0, "bytes": 0, "h2d": 0, "d2h": 0, "e_ms": [], "f_ms": []}
        start.wait()
        torch.cuda.nvtx.range_push("e2e")       # ncu --nvtx-include "e2e/" profiles these
        for s in range(args.steps):
            ih = idx_host[(args.warmup + s) % len(idx_host)]
            with torch.cuda.stream(self.stream):
                self.flush.zero_()
            self.stream.synchronize()
            t1 = time.perf_counter()
            self.table.gather_host(ih, out_host=out_host, stream=self.stream)
            r["e_ms"].append((time.perf_counter() - t1) * 1e3)
            r["e_sec"] += r["e_ms"][-1] / 1e3
            r["bytes"] += ih.numel() * rb
            r["h2d"] += ih.numel() * 8
            r["d2h"] += ih.numel() * rb
        torch.cuda.nvtx.range_pop()
        start.wait()
        for s in range(args.steps):
            ih = idx_host[(args.warmup + s) % len(idx_host)]
            with torch.cuda.stream(self.stream):
                self.flush.zero_()
            self.stream.synchronize()
            t1 = time.perf_counter()
            with torch.cuda.stream(self.stream):
                idx_d = self.idx_up[: ih.numel()]
                idx_d.copy_(ih, non_blocking=True)
                res = self.table.gather(idx_d, out=self.out[: ih.numel() * rb], stream=self.stream)
                probe.copy_(res[:8].view(torch.int64), non_blocking=True)
            self.stream.synchronize()
            r["f_ms"].append((time.perf_counter() - t1) * 1e3)
            r["f_sec"] += r["f_ms"][-1] / 1e3
        del out_host, idx_host
        return r


class StubWorker:
    """--dry-run stand-in for BoxWorker (no GPU, no library): numpy row copies timed on the host,
    so the harness's launch, threading and reductions are testable on CPU. Its numbers are not
    a measurement of anything."""

    def __init__(self, g, table_view, spec, lists, args):
        self.g, self.view, self.spec, self.lists, self.args = g, table_view, spec, lists, args
        self.rb = spec["row_bytes"]

    def gather(self, k):
        l = self.lists[k % len(self.lists)]
        np.take(self.view, l, axis=0)
        return l.size * self.rb

    def warmup(self):
        for s in range(self.args.warmup):
            self.gather(s)

    def timed(self, start):
        start.wait()
        t0 = time.perf_counter()
        ms, nbytes = [], 0
        for s in range(self.args.steps):
            t1 = time.perf_counter()
            nbytes += self.gather(self.args.warmup + s)
            ms.append((time.perf_counter() - t1) * 1e3)
        return {"bytes": nbytes, "ms": ms, "wall_s": time.perf_counter() - t0}


def run_box(args, spec, dist=None):
    """The default harness (any N): ONE process drives all N GPUs, one host thread each, over ONE
    host table (the paper's managed unified tensor, `box_table`). Each GPU gathers its own
    minibatch stream (GPU g takes the rank-g slices of the seeded roots): data parallel by
    minibatch with no collective on the path ("scaling": "weak"). value = Σ_g useful
    bytes ÷ max_g (summed per-step device time)."""
    N = args.gpus
    seed = args.seed
    count = min(args.warmup + args.steps, args.max_lists)
    procs = max(1, (os.cpu_count() or 1) // max(1, min(N, 4)))
    lists = [make_index_lists(spec, g, N, count, seed, procs) for g in range(N)]  # before CUDA
    if args.presort:   # experiment only: what a perfectly address-ordered list would give
        lists = [[np.sort(l) for l in ls] for ls in lists]
    timed_lists = [lists[0][(args.warmup + s) % count] for s in range(args.steps)]
    if args.dry_run:
        rows, rb = spec["rows"], spec["row_bytes"]
        view = np.zeros((min(rows, 1 << 16), rb), dtype=np.uint8)
        lists = [[l % view.shape[0] for l in ls] for ls in lists]
        workers = [StubWorker(g, view, spec, lists[g], args) for g in range(N)]
        run_threads(N, lambda g: workers[g].warmup())
        start = threading.Barrier(N)
        res = run_threads(N, lambda g: workers[g].timed(start))
        dev_ms = [sum(r["ms"]) for r in res]
        total = sum(r["bytes"] for r in res)
        value = total / (max(dev_ms) / 1e3) / 1e9
        if dist is not None and dist.world > 1:       # the launch check: every rank is present
            ranks = int(dist.allreduce([1.0], "sum")[0])
        else:
            ranks = 1
        print(json.dumps({
            "metric": METRIC, "value": round(value, 6), "unit": "GB/s", "n_gpus": N,
            "steps": args.steps, "warmup": args.warmup, "dry_run": True,
            "harness": "threads (one process, one thread per GPU)", "launcher_ranks": ranks,
            "ms_per_step": round(max(dev_ms) / args.steps, 6),
            "per_gpu": [{"gpu": g, "bytes": r["bytes"], "ms": round(sum(r["ms"]), 6)}
                        for g, r in enumerate(res)],
            "config": {"workload": spec["workload"], "seed": seed},
            "note": "--dry-run: numpy stand-in for the GPU arm, NOT a measurement"}), flush=True)
        return

    import torch
    ndev = torch.cuda.device_count()
    if ndev < N and not args.oversubscribe:
        raise SystemExit(f"--gpus {N}: only {ndev} CUDA device(s) visible")
    dev_of = (lambda g: g % ndev) if args.oversubscribe else (lambda g: g)
    torch.cuda.set_device(0)
    import paper_2101_07956_b200 as ut
    t_reg = time.perf_counter()
    tables, owners, kind = box_table(spec, args, ut)
    table, hb = tables[0], owners[0]
    rep = [replica_of(dev_of(g), g, len(tables)) for g in range(N)]
    reg_s = time.perf_counter() - t_reg
    if args.plan:
        for p in args.plan.split(","):
            for tb in tables:
                tb.set_plan(p)
    rb = spec["row_bytes"]
    samplers = None
    if args.sample == "gpu":
        # GPU-side neighbour sampling on every GPU from ONE host CSR: each worker
        # samples its own roots' minibatch, then gathers it (sync mode: one count read per step)
        assert not (args.pipeline and args.coop != "off"), "--pipeline with --coop: not supported"
        csr = workloads.CSRGraph(spec["rows"], spec["edges"], seed=seed, threads=0)

        def mk_sampler(g):
            torch.cuda.set_device(dev_of(g))
            return GpuSampling(spec, g, N, count, seed, ut, torch, args.graph_indptr, "sync",
                               csr=csr)
        samplers = run_threads(N, mk_sampler)
        lists = run_threads(N, lambda g: (torch.cuda.set_device(dev_of(g)),
                                          samplers[g].node_lists_for_accounting())[1])
        timed_lists = [lists[0][(args.warmup + s) % count] for s in range(args.steps)]
    workers = run_threads(N, lambda g: BoxWorker(dev_of(g), torch, tables[rep[g]], spec, lists[g], args))
    if samplers is not None:
        for g in range(N):
            workers[g].sampler = samplers[g]
    coops = None
    if args.coop == "device":
        # the cooperative gather among this process's GPUs (ut_coop_open_local):
        # each row requested by several GPUs in a step is fetched from the host table once, by
        # its owner, and exchanged over NVLink peer memory
        max_n = max(l.size for ls in lists for l in ls)
        if samplers is not None:          # a sampled minibatch may reach the sampler's bound
            max_n = max(smp.capacity() for smp in samplers)

        def mk(g):
            torch.cuda.set_device(dev_of(g))
            return ut.Coop(tables[rep[g]], max_n, rank=g, world=N, sync="device", local=True)
        coops = run_threads(N, mk)
        run_threads(N, lambda g: (torch.cuda.set_device(dev_of(g)), coops[g].open_local(coops)))
        for g in range(N):
            workers[g].coop = coops[g]
            if samplers is not None:      # the sampled rows go through the cooperative gather
                samplers[g].gather_fn = (lambda c: lambda nodes, o: c.gather(nodes, out=o))(coops[g])

    # roofline denominators, measured now: each GPU's link alone, then all at once
    ndevs = len({dev_of(g) for g in range(N)})

    def link(g, reps=10):
        torch.cuda.set_device(dev_of(g))
        return h2d_ceiling(torch, stream=workers[g].stream, reps=reps)
    link_solo = [link(g) for g in range(ndevs)]
    link_nodes = []
    for g in range(ndevs):
        torch.cuda.set_device(dev_of(g))
        link_nodes.append(h2d_ceiling_by_node(torch, dev_of(g)))
    link_conc = run_threads(ndevs, link) if ndevs > 1 else list(link_solo)
    topo = box_topology(torch, sorted({dev_of(g) for g in range(N)}))
    torch.cuda.set_device(0)
    sm_ceiling = sm_read_ceiling(torch, ut)

    parity_lists = 0
    if args.check:
        budget = (16 << 30) // N
        if coops is not None:     # every rank takes part in every cooperative step
            budget = 0            # -> exactly two lists on every GPU
        parity_lists = sum(run_threads(N, lambda g: (torch.cuda.set_device(dev_of(g)),
                                                      workers[g].parity(owners[rep[g]].addr, budget))[1]))

    clocks = ClockSampler(sorted({dev_of(g) for g in range(N)}))
    clocks.start()
    run_threads(N, lambda g: (torch.cuda.set_device(dev_of(g)), workers[g].warmup()))
    for tb in tables:
        tb.set_plan("timing=on")
    devices = sorted({dev_of(g) for g in range(N)})

    def dev_stats():      # the library counts per table and device
        out = []
        for d in devices:
            torch.cuda.set_device(d)
            out.extend(tb.stats(reset=True) for tb in tables)
        return out
    dev_stats()
    coop0 = [c.stats() for c in coops] if coops is not None else None
    if samplers is not None:
        for smp in samplers:
            smp.mark()
    start = threading.Barrier(N)
    gc.collect()
    gc.disable()          # no collector pauses inside the timed host loops
    clocks.mark(0)
    res = run_threads(N, lambda g: (torch.cuda.set_device(dev_of(g)), workers[g].timed(start))[1])
    clocks.mark(1)
    gc.enable()
    clk = clocks.stop()
    stats = dev_stats()
    for tb in tables:
        tb.set_plan("timing=off")
    # the link ceiling again, right after timing: box drift shows as a change here
    link_after = run_threads(ndevs, lambda g: link(g, reps=5)) if ndevs > 1 else [link(0, reps=5)]

    dev_ms = [sum(r["ms"]) for r in res]
    total = sum(r["bytes"] for r in res)
    value = total / (max(dev_ms) / 1e3) / 1e9
    per_gpu = [r["bytes"] / (m / 1e3) / 1e9 for r, m in zip(res, dev_ms)]
    kern_ms = sum(s["gather_kernel_ms"] for s in stats)
    kern_n = sum(s["timed_launches"] for s in stats)
    # per GPU: all GPUs' useful bytes over the sum of their gather-kernel durations
    kern_bytes = total
    launches = sum(s["kernel_launches"] for s in stats)
    if coops is not None:   # the gather kernels fetch the owners' unique rows only
        coop1 = [c.stats() for c in coops]
        kern_bytes = sum(b["unique_rows_fetched"] - a["unique_rows_fetched"]
                         for a, b in zip(coop0, coop1)) * rb
        launches += sum(b["kernel_launches"] - a["kernel_launches"] for a, b in zip(coop0, coop1))
    if samplers is not None:
        launches += sum(smp.timed_launches(args.steps) for smp in samplers)
    achieved = kern_bytes / (kern_ms / 1e3) / 1e9 if kern_ms > 0 else None
    shared = any(s.get("share_gathers") for s in stats)
    plan_label = table.plan + ("+share" if shared else "")
    all_ms = [m for r in res for m in r["ms"]]

    coop_block = None
    if coops is not None:
        cs = [c.stats() for c in coops]
        req = sum(c["requested_rows"] for c in cs)
        uniq = sum(c["unique_rows_fetched"] for c in cs)
        coop_block = {"sync": "device (in-process ranks, ut_coop_open_local)", "ranks": N,
                      "requested_rows_all_steps": req, "host_rows_all_steps": uniq,
                      "host_bytes_fraction": round(uniq / max(1, req), 4),
                      "note": "counters cover parity, warm-up and timed steps; value counts useful "
                              "rows (n*rb per GPU), the host link moved host_bytes_fraction of them"}
    e2e = None
    if not args.no_e2e and coops is None and samplers is None:
        start = threading.Barrier(N)
        gc.collect()
        gc.disable()
        er = run_threads(N, lambda g: (torch.cuda.set_device(dev_of(g)), workers[g].e2e(start))[1])
        gc.enable()
        if os.environ.get("UT_BENCH_DEBUG"):
            for g, r in enumerate(er):
                print(f"e2e gpu{g} host->host ms: {[round(x, 3) for x in r['e_ms']]}", file=sys.stderr)
                print(f"e2e gpu{g} to_hbm ms: {[round(x, 3) for x in r['f_ms']]}", file=sys.stderr)
        eb = sum(r["bytes"] for r in er)
        e2e = {"value": round(eb / max(r["e_sec"] for r in er) / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": int(sum(r["h2d"] for r in er) / args.steps),
               "d2h_bytes_per_step": int(sum(r["d2h"] for r in er) / args.steps),
               "path": "ut_gather_host on every GPU at once: pinned host idx in, pinned host rows out",
               "step_ms": step_stats([m for r in er for m in r["e_ms"]]),
               "to_hbm": {"value": round(eb / max(r["f_sec"] for r in er) / 1e9, 3), "unit": "GB/s",
                          "h2d_bytes_per_step": int(sum(r["h2d"] for r in er) / args.steps),
                          "d2h_bytes_per_step": 8 * N,
                          "step_ms": step_stats([m for r in er for m in r["f_ms"]]),
                          "path": "Table.gather with a pinned host idx: idx H2D, gather into HBM, "
                                  "8-B read-back of the result (the paper's Listing 2 pipeline)"}}

    # NCCL all-reduce smoke (N > 1, untimed, off the gather path; SURVEY §2.3 ii): one
    # single-process multi-GPU all-reduce over NVLink/NVSwitch
    ar = None
    if N > 1 and not args.no_allreduce_smoke and not args.oversubscribe:
        try:        # context, off the measured path: a failure is reported, not fatal
            import torch.cuda.nccl as nccl
            bufs = []
            for g in range(N):
                with torch.cuda.device(g):
                    bufs.append(torch.full((1 << 20,), float(g + 1), dtype=torch.float32,
                                           device="cuda"))
            t1 = time.perf_counter()
            nccl.all_reduce(bufs)
            for g in range(N):
                torch.cuda.synchronize(g)
            want = N * (N + 1) / 2
            ar = {"ok": all(bool((b == want).all().item()) for b in bufs),
                  "bytes": bufs[0].numel() * 4, "ms": round((time.perf_counter() - t1) * 1e3, 3),
                  "backend": "nccl (torch.cuda.nccl, one process, all GPUs)", "gpus": N}
            del bufs
        except Exception as e:  # noqa: BLE001
            ar = {"ok": False, "error": f"{type(e).__name__}: {e}"[:300]}

    dram = None
    if not args.no_cpu:
        import baselines
        dram = round(baselines.host_read_gbs(hb.addr, min(spec["rows"] * rb, 8 << 30)), 2)
    cpu_base, py_base = None, None
    if N == 1 and not args.no_cpu:
        torch.cuda.set_device(0)
        v, nl, el = cpu_oracle_rate(hb.addr, spec, lists[0], args.cpu_budget)
        cpu_base = {"value": round(v, 4), "unit": "GB/s", "cores": 1, "cpu_model": cpu_model(), "kind": "oracle",
                    "sample": f"{nl} minibatches of the workload in {el:.1f} s, single-threaded plain C",
                    "pinned_cpu": getattr(cpu_oracle_rate, "pinned_cpu", None)}
        py_base = cpu_staged_baseline(torch, hb.addr, spec, lists[0], args)
        py_base.pop("_raw", None)
    elif N > 1 and not args.no_cpu and coops is None and samplers is None:
        py_base = cpu_staged_box(torch, run_threads, N, lambda g: owners[rep[g]].addr, spec, lists,
                                 args, lambda g: torch.cuda.set_device(dev_of(g)))

    cfg = config_block(spec, timed_lists, N, seed)
    if samplers is not None and args.pipeline:
        cfg["l2"] = "not flushed: sampling k+1 overlaps gathering k in one timed region (each step writes > L2)"
    sect_ratio = (cfg["sector_floor_mb_per_step"] / cfg["mb_per_step_per_gpu"]
                  if cfg.get("mb_per_step_per_gpu") else None)
    link_g = statistics.mean(link_solo)
    box_link = sum(link_conc)
    ncu_rec = ncu_traffic(spec["workload"], plan_label, kind, args)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": "GB/s", "n_gpus": N,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(max(dev_ms) / args.steps, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic (self-identifying fp32-row table, GraphSAGE-shaped index lists)",
        "config": cfg,
        "harness": "threads: one process drives all GPUs (one host thread each) over one table"
                   + (f" (--oversubscribe: {N} workers on {ndev} device(s), a harness test, not "
                      f"a scaling measurement)" if args.oversubscribe and ndev < N else ""),
        "step_ms": (step_stats(all_ms) if not (samplers is not None and args.pipeline) else
                    {"note": "--pipeline: one timed region per GPU for all K steps",
                     "region_ms": [round(m, 4) for m in all_ms]}),
        "per_gpu_gbs": [round(x, 3) for x in per_gpu],
        "transferred_gbs_sector_floor": round(value * sect_ratio, 3) if sect_ratio else None,
        **transferred_ncu(value, ncu_rec),
        "line_requests_per_s": (round(cfg["line_requests_per_step"] * N / (max(dev_ms) / args.steps / 1e3))
                                if cfg.get("line_requests_per_step") else None),
        "h2d_memcpy_gbs": round(link_g, 3),
        "h2d_memcpy_gbs_per_gpu": [round(x, 3) for x in link_solo],
        "h2d_memcpy_concurrent_gbs": round(box_link, 3),
        "host_links": topo,
        "h2d_memcpy_gbs_by_numa_node": (link_nodes if any(x is not None for x in link_nodes) else
                                        "one NUMA node: the same as h2d_memcpy_gbs"),
        "h2d_memcpy_gbs_after_timing": [round(x, 3) for x in link_after],
        "host_dram_read_gbs": dram,
        "box_roofline_gbs": round(min(box_link, dram), 3) if dram else round(box_link, 3),
        "frac_of_link": round(value / N / link_g, 4),
        "frac_of_box_roofline": round(value / (min(box_link, dram) if dram else box_link), 4),
        "sm_read_ceiling_gbs": round(sm_ceiling, 3),
        "frac_of_sm_read_ceiling": round(value / N / sm_ceiling, 4),
        "plan": plan_label,
        "table_memory": kind + ((f" (cudaMallocManaged + SetPreferredLocation=CPU + SetAccessedBy "
                                 f"every GPU: {len(tables)} replicas, one per NUMA node)") if len(tables) > 1
                                else " (cudaMallocManaged + SetPreferredLocation=CPU + SetAccessedBy "
                                     "every GPU: one copy for the box)" if kind == "managed" else ""),
        "numa": ({"nodes": workloads.numa_nodes(),
                  "policy": f"one replica per node ({len(tables)} tables, {len(tables)}x the host "
                            f"memory; SURVEY §8e)", "replicas": [o.numa for o in owners],
                  "gpu_replica": rep} if len(tables) > 1 else
                 {"nodes": workloads.numa_nodes(),
                  **(hb.numa if isinstance(getattr(hb, "numa", None), dict) else
                     {"policy": "mbind interleave" if getattr(hb, "numa", 0) > 1 else "first touch"})}),
        "roofline": {"bound": "pcie_h2d",
                     "achieved": round(achieved, 3) if achieved is not None else None,
                     "peak": round(link_g, 3), "unit": "GB/s",
                     "frac": round(achieved / link_g, 4) if achieved is not None else None,
                     **ncu_rec,
                     "kernel": f"gather {plan_label} (device time of the gather kernels, share "
                               f"hash/mark included, CUDA events on the launch stream; per GPU)",
                     "timed_launches": kern_n,
                     "peak_source": "pinned cudaMemcpy H2D measured in this run (best of 10 x 1 GiB), "
                                    "mean over the GPUs, each alone",
                     "sm_read_ceiling": round(sm_ceiling, 3)},
        "cpu_baseline": cpu_base, "py_baseline": py_base, "e2e": e2e,
        "gpu_launches": int(launches), "clocks": clk,
        "parity_checked": bool(args.check), "parity_lists_checked": parity_lists,
        "register_s": round(reg_s, 3), "allreduce_smoke": ar, "coop": coop_block,
        "sampling": samplers[0].report(args.steps) if samplers is not None else None,
        "wall_ms_per_step": round(max(r["wall_s"] for r in res) / args.steps * 1e3, 3),
    }
    print(json.dumps(line), flush=True)
    if coops is not None:
        for g in range(N):
            torch.cuda.set_device(dev_of(g))
            torch.cuda.synchronize()
        for g in range(N):
            torch.cuda.set_device(dev_of(g))
            coops[g].close()
            workers[g].coop = None
    del workers
    for tb, o in zip(tables, owners):
        tb.close()
        o.close()


class GpuSampling:
    """`--sample gpu`: every step samples its minibatch on the GPU from a host-resident CSR graph
    (ut_sample) and gathers the rows of the sampled nodes — the whole minibatch
    preparation with no CPU in the loop. The CSR is an explicit Chung-Lu graph of the config's
    N and E (workloads.CSRGraph); each step's 'batch' roots are the rank's slice of a seeded
    permutation."""

    def __init__(self, spec, rank, world, count, seed, ut, torch, indptr="host", mode="sync",
                 csr=None):
        assert spec["kind"] == "graphsage", "--sample gpu needs a graphsage-shaped config"
        self.torch, self.ut, self.spec = torch, ut, spec
        # csr: one host CSR shared by the box harness's GPU workers (each registers it itself)
        self.csr = csr if csr is not None else workloads.CSRGraph(spec["rows"], spec["edges"],
                                                                   seed=seed, threads=0)
        self.graph = ut.Graph(self.csr.indptr_addr, self.csr.indices_addr, self.csr.n_nodes,
                              self.csr.n_edges, keep=self.csr)
        for opt in indptr.split(","):
            self.graph.set_option(f"indptr={opt}" if opt in ("host", "hbm") else opt)
        self.indptr = indptr
        perm = np.random.default_rng(seed + 99).permutation(spec["rows"])
        B = spec["batch"]
        self.roots = [perm[((b * world + rank) * B) % spec["rows"]:][:B].astype(np.int64)
                      for b in range(count)]
        self.roots_dev = [torch.from_numpy(r).cuda() for r in self.roots]
        self.fanouts = list(spec["fanouts"])
        self.seed = seed
        cap = B
        for f in self.fanouts:
            cap += cap * f
        self.nodes = torch.empty(min(cap, spec["rows"]), dtype=torch.int64, device="cuda")
        self.ms_sample, self.rows, self.mid = 0.0, 0, []
        self.mode = mode
        self.seeds_buf = torch.empty(B, dtype=torch.int64, device="cuda")
        self.n_dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.counts = torch.zeros(4096, dtype=torch.int64, device="cuda")
        self.k = 0
        self.cuda_graph = None
        self.graph_kernels = 0
        self._l_mark = 0
        self.gather_fn = None      # --coop: the cooperative gather replaces table.gather (sync mode)

    def capacity(self) -> int:
        return self.nodes.numel()

    def _gather(self, table, nodes, out_view):
        if self.gather_fn is not None:
            self.gather_fn(nodes, out_view)
        else:
            table.gather(nodes, out=out_view)

    def node_lists_for_accounting(self):
        """The minibatches' node lists, computed on the GPU once (for the traffic model and the
        buffer sizes; the timed steps sample again)."""
        out = []
        for b, r in enumerate(self.roots_dev):
            out.append(self.graph.sample(r, self.fanouts, self.seed + b, out=self.nodes).cpu().numpy())
        return out

    def step(self, s, table, out):
        """One minibatch: sample on the GPU, then gather its rows. Synchronous API (one host
        sync per minibatch to learn the count) unless --async-sample: then ut_sample_async +
        ut_gather_dn keep the count on the device (no host sync), optionally replayed from a
        CUDA graph captured once (--graph). Returns rows gathered (host-known modes) or 0."""
        torch = self.torch
        b = s % len(self.roots_dev)
        if self.mode == "sync":
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            nodes = self.graph.sample(self.roots_dev[b], self.fanouts, self.seed + b, out=self.nodes)
            e1.record()
            self.mid.append((e0, e1))
            n = nodes.numel()
            self._gather(table, nodes, out[: n * self.spec["row_bytes"]])
            self.rows += n
            return n
        self.seeds_buf.copy_(self.roots_dev[b])
        if self.mode == "graph":
            if self.cuda_graph is None:
                self._capture(table, out)
            self.cuda_graph.replay()
        else:
            self.graph.sample_async(self.seeds_buf, self.fanouts, self.seed, self.nodes, self.n_dev)
            table.gather_dn(self.nodes, self.n_dev, out)
        self.counts[self.k % self.counts.numel()].copy_(self.n_dev[0])
        self.k += 1
        return 0

    def _capture(self, table, out):
        torch = self.torch
        st = torch.cuda.Stream()
        st.wait_stream(torch.cuda.current_stream())
        self.cuda_graph = torch.cuda.CUDAGraph()
        l0 = self.graph.launches() + table.stats()["kernel_launches"]
        with torch.cuda.graph(self.cuda_graph, stream=st):
            self.graph.sample_async(self.seeds_buf, self.fanouts, self.seed, self.nodes, self.n_dev,
                                    stream=st)
            table.gather_dn(self.nodes, self.n_dev, out, stream=st)
        torch.cuda.current_stream().wait_stream(st)
        self.graph_kernels = self.graph.launches() + table.stats()["kernel_launches"] - l0

    def timed_launches(self, steps) -> int:
        """Sampler kernels in the timed region (graph replays: the captured count x steps)."""
        if self.mode == "graph":
            return self.graph_kernels * steps
        n = self.graph.launches() - self._l_mark
        return n

    def mark(self):
        self._l_mark = self.graph.launches()

    def device_rows(self) -> int:
        """Rows gathered by the device-counted steps since the last call."""
        k = min(self.k, self.counts.numel())
        n = int(self.counts[:k].sum().item())
        self.k = 0
        return n

    def pipelined(self, first, steps, table, out):
        """Steps first..first+steps-1 with sampling of step k+1 overlapping the gather of step k
        (two node buffers, two streams). Returns (useful bytes, elapsed ms on the gather side)."""
        torch = self.torch
        rb = self.spec["row_bytes"]
        ss, sg = torch.cuda.Stream(), torch.cuda.Stream()
        bufs = [self.nodes, torch.empty_like(self.nodes)]
        sampled = [torch.cuda.Event(), torch.cuda.Event()]
        gathered = [torch.cuda.Event(), torch.cuda.Event()]
        start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        nb = len(self.roots_dev)
        with torch.cuda.stream(ss):
            nodes = [self.graph.sample(self.roots_dev[first % nb], self.fanouts,
                                       self.seed + first % nb, out=bufs[0], stream=ss), None]
            sampled[0].record(ss)
        total = 0
        start.record(sg)
        for k in range(steps):
            cur, nxt = k % 2, (k + 1) % 2
            sg.wait_event(sampled[cur])
            n = nodes[cur].numel()
            with torch.cuda.stream(sg):
                table.gather(nodes[cur], out=out[: n * rb], stream=sg)
            gathered[cur].record(sg)
            total += n * rb
            if k + 1 < steps:
                b = (first + k + 1) % nb
                ss.wait_event(gathered[nxt])
                with torch.cuda.stream(ss):
                    nodes[nxt] = self.graph.sample(self.roots_dev[b], self.fanouts, self.seed + b,
                                                   out=bufs[nxt], stream=ss)
                    sampled[nxt].record(ss)
        end.record(sg)
        torch.cuda.synchronize()
        self.rows += total // rb
        return total, start.elapsed_time(end)

    def check(self, table_addr, table, out) -> bool:
        import oracle
        r = self.roots[0]
        want_nodes = oracle.sample(self.csr.indptr_addr, self.csr.indices_addr, self.csr.n_nodes,
                                   r, self.fanouts, self.seed)
        got_nodes = self.graph.sample(self.roots_dev[0], self.fanouts, self.seed, out=self.nodes)
        if not np.array_equal(got_nodes.cpu().numpy(), want_nodes):
            return False
        rb = self.spec["row_bytes"]
        want, _ = oracle.gather(table_addr, self.spec["rows"], rb, want_nodes)
        self._gather(table, got_nodes, out[: got_nodes.numel() * rb])
        return out[: got_nodes.numel() * rb].cpu().numpy().tobytes() == want.tobytes()

    def report(self, steps):
        import time as _t
        import oracle
        self.torch.cuda.synchronize()
        ms = [a.elapsed_time(b) for a, b in self.mid[-steps:]]
        if not ms:      # device-counted modes: time the sampler alone on a few minibatches
            for b in range(min(5, len(self.roots_dev))):
                self.seeds_buf.copy_(self.roots_dev[b])
                e0 = self.torch.cuda.Event(enable_timing=True)
                e1 = self.torch.cuda.Event(enable_timing=True)
                e0.record()
                self.graph.sample_async(self.seeds_buf, self.fanouts, self.seed, self.nodes, self.n_dev)
                e1.record()
                self.torch.cuda.synchronize()
                ms.append(e0.elapsed_time(e1))
        t0 = _t.perf_counter()
        for b in range(3):
            oracle.sample(self.csr.indptr_addr, self.csr.indices_addr, self.csr.n_nodes,
                          self.roots[b], self.fanouts, self.seed + b)
        cpu_ms = (_t.perf_counter() - t0) / 3 * 1e3
        return {"where": "gpu (ut_sample over the host-resident CSR), inside every timed step",
                "graph": f"explicit Chung-Lu CSR, N={self.csr.n_nodes}, E={self.csr.n_edges}",
                "indptr": self.indptr, "mode": self.mode,
                "gpu_sample_ms_per_step": round(float(np.mean(ms)), 3),
                "gpu_sample_ms_measured_on": "timed steps (sync mode) or 5 standalone async samples",
                "oracle_cpu_sample_ms_per_minibatch": round(cpu_ms, 2), "oracle_cores": 1}


def cpu_model() -> str:
    """The host CPU model ("Report T and the CPU model"): the model name, and — since
    virtualised hosts report a generic name — family/model numbers and the L3 size, which decide
    how much of a CPU gather's staging stays in cache."""
    name, fam, mod = "unknown", "?", "?"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                k, _, v = line.partition(":")
                k = k.strip()
                if k == "model name" and name == "unknown":
                    name = v.strip()
                elif k == "cpu family" and fam == "?":
                    fam = v.strip()
                elif k == "model" and mod == "?":
                    mod = v.strip()
                if name != "unknown" and fam != "?" and mod != "?":
                    break
    except OSError:
        pass
    try:
        with open("/sys/devices/system/cpu/cpu0/cache/index3/size") as f:
            l3 = f.read().strip()
    except OSError:
        l3 = "?"
    return f"{name} (family {fam} model {mod}, L3 {l3})"


def cpu_staged_baseline(torch, table_addr, spec, lists, args, threads=None, barrier=None):
    """The paper's "Py" path (Fig. 2a): all host cores gather into pinned
    staging, then one H2D DMA. Three forms: sequential (paper-faithful), double-
    buffered (chunk k+1 gathered while chunk k is in flight: the stronger CPU-centric baseline),
    and pageable (Listing 1 literally, `features[neighbor_id].to("cuda")`, PAPER.md:315-316,
    torch's own CPU index_select into pageable memory). At k GPUs ("T = cores/k per
    rank") one call per GPU runs concurrently with `threads` host threads each, `barrier`
    starting every form on all GPUs together; the raw (bytes, seconds) of each form are returned
    under "_raw" for the box aggregate, and the pageable form is skipped."""
    import baselines
    rb = spec["row_bytes"]
    max_n = max(l.size for l in lists)
    staging = torch.empty(max_n * rb, dtype=torch.uint8, pin_memory=True)
    dev = torch.empty(max_n * rb, dtype=torch.uint8, device="cuda")
    threads = threads or os.cpu_count() or 1
    steps = min(len(lists), max(3, args.steps // 2))
    chunks = 8
    copy_stream = torch.cuda.Stream()

    def sequential(l):
        b = l.size * rb
        baselines.cpu_staged_gather(table_addr, rb, l.ctypes.data, l.size, staging.data_ptr(), threads)
        dev[:b].copy_(staging[:b], non_blocking=True)

    def double_buffered(l):
        # two halves of the staging buffer alternate; chunk c is gathered into half c % 2 once
        # the DMA of chunk c - 2 (same half) has drained
        per = (l.size + chunks - 1) // chunks
        half = ((per * rb + 4095) // 4096) * 4096
        done = [None, None]
        for c in range(chunks):
            lo, hi = c * per, min(l.size, (c + 1) * per)
            if lo >= hi:
                break
            h = c % 2
            if done[h] is not None:
                done[h].synchronize()
            baselines.cpu_staged_gather(table_addr, rb, l.ctypes.data + 8 * lo, hi - lo,
                                        staging.data_ptr() + h * half, threads)
            with torch.cuda.stream(copy_stream):
                dev[lo * rb:hi * rb].copy_(staging[h * half:h * half + (hi - lo) * rb], non_blocking=True)
                done[h] = torch.cuda.Event()
                done[h].record(copy_stream)
        copy_stream.synchronize()

    buf = (ctypes.c_uint8 * (spec["rows"] * rb)).from_address(table_addr)
    table_view = torch.frombuffer(buf, dtype=torch.uint8).view(spec["rows"], rb)

    def pageable(l):
        table_view[torch.from_numpy(l)].to("cuda")

    raw = {}

    def rate(fn, name):
        sec, nbytes = 0.0, 0
        if barrier is not None:
            torch.cuda.synchronize()
            barrier.wait()
        for s in range(steps + 1):
            l = lists[s % len(lists)]
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn(l)
            torch.cuda.synchronize()
            if s > 0:
                sec += time.perf_counter() - t0
                nbytes += l.size * rb
        raw[name] = (nbytes, sec)
        return round(nbytes / sec / 1e9, 3)

    out = {"value": rate(sequential, "sequential"), "unit": "GB/s", "threads": threads,
           "cpu_model": cpu_model(),
           "kind": "CPU gather into pinned staging + cudaMemcpyAsync H2D (PAPER.md:221-225)",
           "steps": steps, "double_buffered": rate(double_buffered, "double_buffered"),
           "double_buffered_chunks": chunks}
    if barrier is None:
        out["pageable"] = rate(pageable, "pageable")
        out["pageable_kind"] = "torch CPU index_select + pageable .to('cuda') (Listing 1, PAPER.md:315-316)"
    out["_raw"] = raw
    return out


def cpu_staged_box(torch, run_threads_fn, n, addr_of, spec, lists, args, set_dev):
    """SURVEY §8d's CPU-centric baseline at k = n GPUs: every GPU's Py path at once, cores/k host
    threads each; value = Σ bytes ÷ max seconds per form, with the per-GPU rates beside it."""
    import baselines
    baselines.lib()
    per = max(1, (os.cpu_count() or 1) // n)
    bar = threading.Barrier(n)
    res = run_threads_fn(n, lambda g: (set_dev(g), cpu_staged_baseline(
        torch, addr_of(g), spec, lists[g], args, threads=per, barrier=bar))[1])

    def agg(name):
        b = sum(r["_raw"][name][0] for r in res)
        sec = max(r["_raw"][name][1] for r in res)
        return round(b / sec / 1e9, 3)
    return {"value": agg("sequential"), "unit": "GB/s", "gpus": n, "threads_per_gpu": per,
            "cpu_model": cpu_model(),
            "kind": "CPU gather into pinned staging + cudaMemcpyAsync H2D (PAPER.md:221-225), "
                    "every GPU at once, cores/k threads per GPU (SURVEY §8d)",
            "double_buffered": agg("double_buffered"),
            "per_gpu_sequential": [r["value"] for r in res],
            "per_gpu_double_buffered": [r["double_buffered"] for r in res],
            "steps": res[0]["steps"], "double_buffered_chunks": res[0]["double_buffered_chunks"]}


def self_launch(args, argv) -> int:
    """`--harness procs` at N > 1 without torchrun: start the N ranks ourselves (torchrun on
    127.0.0.1, one process per GPU) and return their exit code."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port",
           str(port), os.path.abspath(__file__), *argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = list(sys.argv[1:] if argv is None else argv)
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="papers",
                    help="papers (default: ogbn-papers100M-shaped, the largest single-GPU config), "
                         "products, reddit, tiny, sweep:RB")
    ap.add_argument("--impl", default="ut", choices=["ut", "reference"])
    ap.add_argument("--harness", default="threads", choices=["threads", "procs"],
                    help="threads (default): one process drives all N GPUs over one table; "
                         "procs: one process per GPU (torchrun ranks; --coop, --sample gpu)")
    ap.add_argument("--dry-run", action="store_true",
                    help="harness test without a GPU: numpy stand-in for the GPU arm")
    ap.add_argument("--oversubscribe", action="store_true",
                    help="harness test: GPU worker g runs on device g %% device_count (N workers "
                         "on fewer GPUs); no all-reduce smoke")
    ap.add_argument("--seed", type=int, default=2101)
    ap.add_argument("--plan", default="", help="comma list passed to ut_set_plan (A/B runs)")
    ap.add_argument("--max-lists", type=int, default=64, help="distinct minibatches per rank")
    ap.add_argument("--cpu-budget", type=float, default=10.0, help="seconds of oracle timing")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", dest="check", action="store_false")
    ap.add_argument("--backend", default="nccl", help="process-group backend at N > 1")
    ap.add_argument("--presort", action="store_true", help="experiment: sort index lists on the host")
    ap.add_argument("--graph-edges", type=int, default=0,
                    help="override Table 4's edge count of a GraphSAGE config (e.g. reddit 114600000)")
    ap.add_argument("--coop", default="off", choices=["off", "device", "host"],
                    help="cooperative gather across ranks (ut_coop; DESIGN.md §10d): phases "
                         "synchronised on the device or by host barriers (implies --harness procs)")
    ap.add_argument("--alloc", default="auto", choices=["auto", "register", "pinned", "managed", "vmm"],
                    help="table memory: auto = managed (the paper's unified tensor) in the threads "
                         "harness; in procs: managed for one rank and a table > 1 GiB, else register")
    ap.add_argument("--numa", default="auto", choices=["auto", "interleave", "replica", "off"],
                    help="threads harness, managed table: stripe its pages over the host NUMA nodes "
                         "(auto: when the box has more than one node), or one replica per node "
                         "(replica: each GPU reads the copy on its own node, if RAM allows)")
    ap.add_argument("--numa-replicas", type=int, default=0,
                    help="--numa replica: number of replicas (0 = one per NUMA node; more than the "
                         "node count places them round-robin — a harness test on one-node boxes)")
    ap.add_argument("--sample", default="cpu", choices=["cpu", "gpu"],
                    help="cpu: index lists sampled before timing (default, the paper's split); "
                         "gpu: ut_sample inside every timed step (SURVEY NEXT-2; implies --harness procs)")
    ap.add_argument("--graph-indptr", default="host",
                    help="with --sample gpu: 'host' or 'hbm' for indptr, optionally ',indices=hbm'")
    ap.add_argument("--async-sample", action="store_true",
                    help="with --sample gpu: ut_sample_async + ut_gather_dn (no host sync)")
    ap.add_argument("--graph", action="store_true",
                    help="with --sample gpu: capture sample + gather once in a CUDA graph, replay")
    ap.add_argument("--pipeline", action="store_true",
                    help="with --sample gpu: sample minibatch k+1 while gathering minibatch k")
    ap.add_argument("--reverse-fanouts", action="store_true",
                    help="graphsage configs: apply the fanouts in reverse hop order (SURVEY c15)")
    ap.add_argument("--allreduce-smoke", action="store_true",
                    help="procs harness, N > 1: one untimed NCCL all-reduce after timing")
    ap.add_argument("--no-allreduce-smoke", action="store_true",
                    help="threads harness: skip the untimed NCCL all-reduce smoke at N > 1")
    args = ap.parse_args(argv)
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if args.coop == "host" or (args.sample != "cpu" and (args.async_sample or args.graph)):
        args.harness = "procs"
    if args.coop == "device" and args.harness == "threads":
        # in-process ranks wait for each other on the device (ut_coop_open_local): one hardware
        # queue per stream when several ranks share a device (--oversubscribe), set before any
        # CUDA context; the kernels a step launches are loaded before the first step (the
        # library's own in ut_coop_open_local, torch's L2 flush in BoxWorker.__init__)
        os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
    spec = workload_spec(args.config)
    if args.reverse_fanouts and spec["kind"] == "graphsage":
        spec["reverse_fanouts"] = True          # DGL's order: the last fanout at the seeds (c15)
        spec["fanouts"] = list(reversed(spec["fanouts"]))
    if args.graph_edges and spec["kind"] == "graphsage":
        spec["edges"] = args.graph_edges        # E sensitivity (reading c17)
    dist = Dist()
    if dist.world > 1 and dist.world != args.gpus:
        raise SystemExit(f"launched with WORLD_SIZE={dist.world} but --gpus {args.gpus}")
    if dist.world == 1 and args.gpus > 1 and args.harness == "procs" and args.impl == "ut":
        return self_launch(args, argv)
    try:
        if args.impl == "reference":
            run_reference(args, spec, dist)
        elif args.harness == "procs":
            run_procs(args, spec, dist)
        elif dist.world > 1:
            # launched by torchrun (one rank per GPU): rank 0 is the box process and drives every
            # GPU over the one table; the other ranks only rendezvous (CPU gloo, no CUDA context)
            dist.init("gloo")
            if dist.rank == 0:
                run_box(args, spec, dist)
            elif args.dry_run:
                dist.allreduce([1.0], "sum")
            dist.barrier()
        else:
            run_box(args, spec)
    finally:
        dist.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
