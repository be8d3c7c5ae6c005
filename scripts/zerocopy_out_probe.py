"""Experiment: gather with idx and/or out in pinned HOST memory (zero-copy), vs device (dev aid)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2101_07956_b200 as ut
import workloads

tbytes = 1 << 30
hb = workloads.HostBuffer(tbytes)
workloads.fill_table(hb.addr, tbytes // 4096, 4096, 1)
n = 400_000
for rb in [400, 512, 2408, 68]:
    rows = tbytes // rb
    idx_h = torch.from_numpy(workloads.uniform_idx(n, rows, rb)).pin_memory()
    idx_d = idx_h.cuda()
    out_d = torch.empty(n * rb, dtype=torch.uint8, device="cuda")
    out_h = torch.empty(n * rb, dtype=torch.uint8, pin_memory=True)
    with ut.Table(hb.addr, rows, rb) as t:
        for name, i, o in [("dev_idx,dev_out", idx_d, out_d), ("host_idx,dev_out", idx_h, out_d),
                           ("dev_idx,host_out", idx_d, out_h), ("host_idx,host_out", idx_h, out_h)]:
            ts = []
            for r in range(5):
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ut.ut_gather(t.handle, i.data_ptr(), n, o.data_ptr(), torch.cuda.current_stream().cuda_stream)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = sorted(ts)[2]
            ok = bool((o[: 64].cpu() == out_d[:64].cpu()).all()) if name != "dev_idx,dev_out" else True
            print(json.dumps({"rb": rb, "mode": name, "gbs": round(n * rb / ms / 1e6, 2), "ok": ok}), flush=True)
