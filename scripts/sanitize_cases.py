"""Tiny cases for compute-sanitizer (memcheck / racecheck / synccheck): every kernel family,
the reorder stage, run merge, neighbour line sharing, the TMA bulk plan, the paper's kernels, host end-to-end, int32 ids, GPU sampling and
the cooperative gather (one rank: dispatch, dedup, host fetch, combine)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import paper_2101_07956_b200 as ut
import workloads

bad = 0
for rb, off in [(4, 0), (8, 8), (68, 3), (400, 0), (400, 4), (144, 0), (2052, 1), (4096, 0), (13, 5)]:
    rows = 3000
    hb = workloads.HostBuffer(rows * rb, kind="guarded")
    workloads.fill_table(hb.addr, rows, rb, rb)
    idx = workloads.uniform_idx(700, rows, rb)
    idx[:2] = [0, rows - 1]
    want, _ = oracle.gather(hb.addr, rows, rb, idx)
    with ut.Table(hb.addr, rows, rb) as t:
        for plan in ["auto", "realign", "realignx", "vec16", "vec16x", "narrow", "bulk", "tma4",
                     "paper_naive", "paper_shift"]:
            try:
                t.set_plan(plan)
            except ut.UTError:
                continue
            for reorder in ["reorder=off,runs=off,share=off", "reorder=on,runs=off,share=off",
                            "reorder=on,runs=off,share=off,exact=on",
                            "reorder=off,runs=on,share=off,exact=off", "reorder=off,runs=off,share=on"]:
                for m in reorder.split(","):
                    t.set_plan(m)
                buf = torch.zeros(700 * rb + 16, dtype=torch.uint8, device="cuda")
                t.gather(torch.from_numpy(idx).cuda(), out=buf[off: off + 700 * rb])
                got = buf[off: off + 700 * rb].cpu().numpy()
                if got.tobytes() != want.tobytes():
                    bad += 1
                    print("MISMATCH", rb, plan, reorder)
        for m in ["auto", "reorder=auto", "runs=auto", "share=auto", "exact=auto"]:
            t.set_plan(m)
        o = t.gather_host(torch.from_numpy(idx).pin_memory())
        bad += o.numpy().tobytes() != want.tobytes()
        o = t.gather(torch.from_numpy(idx.astype(np.int32)).cuda())     # ut_gather_i32
        bad += o.cpu().numpy().tobytes() != want.tobytes()
    hb.close()

g = workloads.CSRGraph(20000, 300000, seed=4)
with ut.Graph(g.indptr_addr, g.indices_addr, g.n_nodes, g.n_edges, keep=g) as gr:
    seeds = np.arange(0, 20000, 97, dtype=np.int64)
    got = gr.sample(torch.from_numpy(seeds).cuda(), [5, 3], 11).cpu().numpy()
    want = oracle.sample(g.indptr_addr, g.indices_addr, g.n_nodes, seeds, [5, 3], 11)
    bad += not np.array_equal(got, want)
for rb, off in [(68, 3), (400, 0), (2408, 8), (13, 1)]:
    rows = 2000
    hb = workloads.HostBuffer(rows * rb, kind="guarded")
    workloads.fill_table(hb.addr, rows, rb, rb + 1)
    idx = workloads.uniform_idx(900, rows, rb + 2)
    idx[:3] = [0, rows - 1, 0]
    idx[7] = rows                      # out of range: zero row + recorded position
    want, want_bad = oracle.gather(hb.addr, rows, rb, idx)
    with ut.Table(hb.addr, rows, rb) as t:
        for sync in ("device", "host"):
            with ut.Coop(t, 1000, world=1, rank=0, sync=sync) as c:
                for _ in range(3):     # both buffer parities
                    buf = torch.zeros(900 * rb + 16, dtype=torch.uint8, device="cuda")
                    c.gather(torch.from_numpy(idx).cuda(), out=buf[off: off + 900 * rb])
                    got = buf[off: off + 900 * rb].cpu().numpy()
                    bad += got.tobytes() != want.tobytes()
                    bad += c.error_pos() != want_bad
    hb.close()
torch.cuda.synchronize()
print("SANITIZE-CASES-DONE bad=%d" % bad)
