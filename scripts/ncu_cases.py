"""One gather launch per case (for ncu metric capture of sysmem/PCIe traffic; dev aid)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2101_07956_b200 as ut
import workloads

CASES = [("seq", 512), ("rand", 512), ("rand", 400), ("rand", 2408), ("rand", 64),
         ("rand", 128), ("rand", 256), ("rand", 4), ("seq", 64), ("sorted", 64)]

tbytes = 1 << 30
hb = workloads.HostBuffer(tbytes)
workloads.fill_table(hb.addr, tbytes // 4096, 4096, 1)
n = 1 << 20
for kind, rb in CASES:
    rows = tbytes // rb
    if kind == "seq":
        idx = np.arange(min(n, rows), dtype=np.int64)
    else:
        idx = workloads.uniform_idx(n, rows, seed=rb)
        if kind == "sorted":
            idx = np.sort(idx)
    idx_d = torch.from_numpy(idx).cuda()
    out = torch.empty(idx.size * rb, dtype=torch.uint8, device="cuda")
    with ut.Table(hb.addr, rows, rb) as t:
        t.set_plan("reorder=off")
        t.gather(idx_d, out=out)
        torch.cuda.synchronize()
        print(json.dumps({"case": kind, "rb": rb, "n": int(idx.size), "plan": t.plan,
                          "useful_bytes": int(idx.size * rb)}), flush=True)
