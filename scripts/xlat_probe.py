"""Experiment: is small-row gather bound by address translation? (development aid)

Sweeps table size, host allocation kind (mmap+THP, mmap 4K, cudaHostAlloc via torch) and index
order (random vs sorted) at a few row widths; prints GB/s and Mrows/s."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2101_07956_b200 as ut
import workloads


def tgather(t, idx_d, out, reps=5):
    ts = []
    for r in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t.gather(idx_d, out=out)
        e1.record()
        torch.cuda.synchronize()
        if r >= 2:
            ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def meminfo(key):
    for l in open("/proc/meminfo"):
        if l.startswith(key):
            return l.split()[1]


def run(kind, gib, widths, n=1 << 20, sort=False):
    tbytes = int(gib * (1 << 30))
    keep = None
    if kind == "cudahost":
        keep = torch.empty(tbytes, dtype=torch.uint8, pin_memory=True)
        addr = keep.data_ptr()
    else:
        keep = workloads.HostBuffer(tbytes, hugepage=(kind == "thp"))
        addr = keep.addr
    arr = (np.ctypeslib.as_array((__import__("ctypes").c_uint8 * tbytes).from_address(addr)))
    workloads.fill_table(arr, tbytes // 4096, 4096, 1)
    res = []
    for rb in widths:
        rows = tbytes // rb
        idx = workloads.uniform_idx(n, rows, seed=rb)
        if sort:
            idx = np.sort(idx)
        idx_d = torch.from_numpy(idx).cuda()
        out = torch.empty(n * rb, dtype=torch.uint8, device="cuda")
        with ut.Table(addr, rows, rb) as t:
            ms = tgather(t, idx_d, out)
        r = {"kind": kind, "gib": gib, "rb": rb, "sorted": sort, "ms": round(ms, 3),
             "gbs": round(n * rb / ms / 1e6, 2), "mrows_s": round(n / ms / 1e3, 1),
             "anon_huge_kb": meminfo("AnonHugePages")}
        print(json.dumps(r), flush=True)
        res.append(r)
    del arr
    if kind != "cudahost":
        keep.close()
    return res


def main():
    print(open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
    widths = [64, 512]
    for gib in [0.0625, 0.25, 1, 4, 16]:
        run("thp", gib, widths)
    run("thp", 4, widths, sort=True)
    run("nothp", 4, widths)
    run("cudahost", 4, widths)
    run("cudahost", 0.25, widths)
    run("cudahost", 4, widths, sort=True)


if __name__ == "__main__":
    main()
