"""Experiment: sorted sparse gathers (papers-like density) vs host allocation kind (dev aid)."""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2101_07956_b200 as ut
import workloads
from xlat_probe import tgather

tbytes = 16 << 30
rb = 512
rows = tbytes // rb
for kind in ["thp", "nothp", "cudahost"]:
    if kind == "cudahost":
        keep = torch.empty(tbytes, dtype=torch.uint8, pin_memory=True)
        addr = keep.data_ptr()
    else:
        keep = workloads.HostBuffer(tbytes, hugepage=(kind == "thp"))
        addr = keep.addr
    workloads.fill_table(addr, tbytes // 4096, 4096, 1)
    with ut.Table(addr, rows, rb) as t:
        t.set_plan("reorder=off")
        for n in [1 << 20, 1 << 18, 1 << 16]:
            idx = np.sort(workloads.uniform_idx(n, rows, seed=n))
            idx_d = torch.from_numpy(idx).cuda()
            out = torch.empty(n * rb, dtype=torch.uint8, device="cuda")
            ms = tgather(t, idx_d, out)
            print(json.dumps({"kind": kind, "n": n, "rows_per_2MB": round(n / (tbytes >> 21), 1),
                              "gbs": round(n * rb / ms / 1e6, 2)}), flush=True)
    if kind != "cudahost":
        keep.close()
    del keep
