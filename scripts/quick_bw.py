"""Quick bandwidth probe (development aid, not the bench): ut_gather GB/s per plan vs H2D memcpy."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2101_07956_b200 as ut
import workloads


def h2d_ceiling(nbytes=1 << 30, reps=10):
    h = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    h.fill_(1)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    best = 0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.copy_(h, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, nbytes / e0.elapsed_time(e1) / 1e6)
    return best


def time_gather(t, idx_d, out, reps=5, flush=None):
    ts = []
    for r in range(reps + 2):
        if flush is not None:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t.gather(idx_d, out=out)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts)), float(min(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--table-gib", type=float, default=4.0)
    ap.add_argument("--n", type=int, default=1 << 20)
    ap.add_argument("--widths", default="4,8,16,64,68,128,256,400,512,1024,2048,2052,2408,4096")
    ap.add_argument("--plans", default="auto")
    args = ap.parse_args()
    ceil = h2d_ceiling()
    print(json.dumps({"h2d_memcpy_gbs": round(ceil, 2)}), flush=True)
    tbytes = int(args.table_gib * (1 << 30))
    hb = workloads.HostBuffer(tbytes + 4096)
    t0 = time.time()
    workloads.fill_table(hb.array()[:tbytes], tbytes // 4096, 4096, 1, threads=0)
    print(json.dumps({"fill_s": round(time.time() - t0, 2)}), flush=True)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rb in [int(x) for x in args.widths.split(",")]:
        rows = tbytes // rb
        n = min(args.n, max(1, (2 << 30) // rb))
        idx = workloads.uniform_idx(n, rows, seed=rb)
        idx_d = torch.from_numpy(idx).cuda()
        out = torch.empty(n * rb, dtype=torch.uint8, device="cuda")
        t1 = time.time()
        t = ut.Table(hb.addr, rows, rb)
        reg_s = time.time() - t1
        for plan in args.plans.split(","):
            try:
                t.set_plan(plan)
            except ut.UTError:
                continue
            med, best = time_gather(t, idx_d, out, flush=flush)
            print(json.dumps({"rb": rb, "plan": t.plan, "n": n, "ms": round(med, 3),
                              "gbs": round(n * rb / med / 1e6, 2),
                              "frac": round(n * rb / med / 1e6 / ceil, 3),
                              "reg_s": round(reg_s, 2)}), flush=True)
        t.close()


if __name__ == "__main__":
    main()
