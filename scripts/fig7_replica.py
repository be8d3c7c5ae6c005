"""Replica of the paper's Fig. 7 microbenchmark on B200 (§5.2).

"The microbenchmark uses a random number generator (RNG) to generate random indices which are
used to index feature values. The total number of items is fixed to 4M" (reading
SURVEY c13: a 4,194,304-row pool). Grid (#rows, row size) from (8K, 256 B) to (256K, 16 KB)
(SPEC.md:426 interior points). For every cell it times, with CUDA events / wall clock:
  * Py   — the CPU-centric path: all host cores gather into pinned staging, then one H2D copy
           (Fig. 2a; baselines/cpu_staged.c);
  * PyD  — this repo's ut_gather (GPU threads read the host table directly);
  * ideal — the bytes at the pinned-memcpy H2D ceiling measured in the same run (the paper's
           'ideal' is the theoretical peak; reading R15).
and prints the paper's figure of merit: slowdown vs ideal (paper: Py 1.85-3.98x, PyD
1.03-1.20x outside (8K, 256 B); PyD over Py 2.39x on average).
Usage: python scripts/fig7_replica.py [--out profiles/r1_fig7_replica.jsonl] [--alloc managed]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import baselines
import paper_2101_07956_b200 as ut
import workloads
from bench import h2d_ceiling

POOL = 4_194_304
ROWS = [8192, 32768, 131072, 262144]
WIDTHS = [256, 1024, 4096, 16384]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="")
    ap.add_argument("--alloc", default="register", choices=["register", "managed"])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--plan", default="", help="comma list for ut_set_plan (A/B)")
    args = ap.parse_args()
    link = h2d_ceiling(torch)
    threads = os.cpu_count() or 1
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    lines = []
    for rb in WIDTHS:
        tbytes = POOL * rb
        if args.alloc == "managed":
            try:
                table = ut.Table.create(POOL, rb, "managed")
            except ut.UTError as e:
                print(json.dumps({"row_bytes": rb, "skipped": f"managed allocation failed: {e}"}))
                continue
            addr = table.host_addr
            hb = None
        else:
            hb = workloads.HostBuffer(tbytes)
            addr = hb.addr
        workloads.fill_table(addr, POOL, rb, rb, threads=0)
        if args.alloc != "managed":
            table = ut.Table(addr, POOL, rb)
        for p in filter(None, args.plan.split(",")):
            table.set_plan(p)
        max_n = max(ROWS)
        staging = torch.empty(max_n * rb, dtype=torch.uint8, pin_memory=True)
        dev = torch.empty(max_n * rb, dtype=torch.uint8, device="cuda")
        for n in ROWS:
            idx = workloads.uniform_idx(n, POOL, seed=n * 7 + rb)
            idx_d = torch.from_numpy(idx).cuda()
            nbytes = n * rb
            # PyD: GPU direct gather
            ts = []
            for r in range(args.reps + 1):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                table.gather(idx_d, out=dev[:nbytes])
                e1.record()
                torch.cuda.synchronize()
                if r:
                    ts.append(e0.elapsed_time(e1) / 1e3)
            pyd = float(np.median(ts))
            # Py: CPU gather into pinned staging + one H2D copy
            ts = []
            for r in range(args.reps + 1):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                baselines.cpu_staged_gather(addr, rb, idx.ctypes.data, n, staging.data_ptr(), threads)
                dev[:nbytes].copy_(staging[:nbytes], non_blocking=True)
                torch.cuda.synchronize()
                if r:
                    ts.append(time.perf_counter() - t0)
            py = float(np.median(ts))
            ideal = nbytes / (link * 1e9)
            rec = {"rows": n, "row_bytes": rb, "mbytes": round(nbytes / 1e6, 1), "table_memory": args.alloc,
                   "pyd_ms": round(pyd * 1e3, 3), "py_ms": round(py * 1e3, 3), "ideal_ms": round(ideal * 1e3, 3),
                   "pyd_slowdown_vs_ideal": round(pyd / ideal, 3), "py_slowdown_vs_ideal": round(py / ideal, 3),
                   "pyd_speedup_over_py": round(py / pyd, 2), "pyd_gbs": round(nbytes / pyd / 1e9, 2),
                   "h2d_memcpy_gbs": round(link, 2), "py_threads": threads, "plan": table.plan}
            print(json.dumps(rec), flush=True)
            lines.append(rec)
        table.close()
        if hb is not None:
            hb.close()
        del staging, dev
    sp = [r["pyd_speedup_over_py"] for r in lines]
    excl = [r for r in lines if not (r["rows"] == 8192 and r["row_bytes"] == 256)]
    summary = {"summary": True, "pyd_slowdown_range": [min(r["pyd_slowdown_vs_ideal"] for r in excl),
                                                       max(r["pyd_slowdown_vs_ideal"] for r in excl)],
               "py_slowdown_range": [min(r["py_slowdown_vs_ideal"] for r in excl),
                                     max(r["py_slowdown_vs_ideal"] for r in excl)],
               "mean_pyd_speedup_over_py": round(float(np.mean(sp)), 2),
               "paper": {"pyd_slowdown": [1.03, 1.20], "py_slowdown": [1.85, 3.98], "mean_speedup": 2.39}}
    print(json.dumps(summary), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            for r in lines + [summary]:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
