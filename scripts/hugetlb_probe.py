"""Experiment: is the ~1-GiB translation reach of registered host memory a page-size effect?
Random 512-B rows (reorder off) over a 16-GiB registered table backed by 4-KiB pages (THP
advised), hugetlbfs 2-MiB pages and 1-GiB pages (reserved here, restored after), vs the managed
allocation. Needs root on the GPU box for /proc/sys/vm/nr_hugepages."""
import ctypes
import json
import mmap
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2101_07956_b200 as ut
import workloads

MAP_HUGETLB = 0x40000
MAP_HUGE_SHIFT = 26
TB = 16 << 30
RB = 512
N = 1 << 20


def sysfs(path, value=None):
    try:
        if value is None:
            return open(path).read().strip()
        with open(path, "w") as f:
            f.write(str(value))
        return open(path).read().strip()
    except OSError as e:
        return f"error: {e}"


def run(name, addr):
    rows = TB // RB
    workloads.fill_table(addr, rows, RB, 1, threads=16)
    idx = torch.from_numpy(workloads.uniform_idx(N, rows, seed=5)).cuda()
    out = torch.empty(N * RB, dtype=torch.uint8, device="cuda")
    t0 = time.perf_counter()
    with ut.Table(addr, rows, RB) as t:
        reg = time.perf_counter() - t0
        for reorder in ("off", "on"):
            t.set_plan(f"reorder={reorder}")
            t.gather(idx, out=out)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(3):
                t.gather(idx, out=out)
            e1.record()
            torch.cuda.synchronize()
            gbs = 3 * N * RB / (e0.elapsed_time(e1) / 1e3) / 1e9
            print(json.dumps({"memory": name, "reorder": reorder, "gbs": round(gbs, 2),
                              "register_s": round(reg, 2)}), flush=True)


def main():
    # 4-KiB pages, THP advised (the default HostBuffer)
    hb = workloads.HostBuffer(TB)
    run("mmap 4K + THP advice", hb.addr)
    hb.close()
    # managed (the paper's allocation)
    t = ut.Table.create(TB // RB, RB, "managed")
    addr = t.host_addr
    workloads.fill_table(addr, TB // RB, RB, 1, threads=16)
    idx = torch.from_numpy(workloads.uniform_idx(N, TB // RB, seed=5)).cuda()
    out = torch.empty(N * RB, dtype=torch.uint8, device="cuda")
    t.set_plan("reorder=off")
    t.gather(idx, out=out); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        t.gather(idx, out=out)
    e1.record(); torch.cuda.synchronize()
    print(json.dumps({"memory": "managed", "reorder": "off",
                      "gbs": round(3 * N * RB / (e0.elapsed_time(e1) / 1e3) / 1e9, 2)}), flush=True)
    t.close()
    del idx, out
    for size_kb, shift, count in ((2048, 21, TB // (2 << 20) + 16), (1048576, 30, TB // (1 << 30) + 1)):
        path = f"/sys/kernel/mm/hugepages/hugepages-{size_kb}kB/nr_hugepages"
        old = sysfs(path)
        got = sysfs(path, count)
        print(json.dumps({"hugepages": size_kb, "requested": count, "reserved": got}), flush=True)
        try:
            m = mmap.mmap(-1, TB, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS | MAP_HUGETLB |
                          (shift << MAP_HUGE_SHIFT))
        except OSError as e:
            print(json.dumps({"hugepages": size_kb, "mmap": f"failed: {e}"}), flush=True)
            sysfs(path, old)
            continue
        addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
        run(f"hugetlbfs {size_kb // 1024} MiB pages", addr)
        del addr
        m.close()
        sysfs(path, old)


if __name__ == "__main__":
    main()
