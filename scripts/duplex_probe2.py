"""Experiment: which direction limits end-to-end? Rates of each stream when overlapped (dev aid)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2101_07956_b200 as ut
import workloads
from paper_2101_07956_b200.unified import _CudaArray

def ev(): return torch.cuda.Event(enable_timing=True)
N = 512 << 20
rows, rb = (1 << 30) // 512, 512
hb = workloads.HostBuffer(rows * rb); workloads.fill_table(hb.addr, rows, rb, 1)
t = ut.Table(hb.addr, rows, rb)
n = N // rb
idx = torch.from_numpy(workloads.uniform_idx(n, rows, 3)).cuda()
gout = torch.empty(N, dtype=torch.uint8, device="cuda")
dsrc = torch.ones(N, dtype=torch.uint8, device="cuda")
hdst = torch.empty(N, dtype=torch.uint8, pin_memory=True)
hview = torch.as_tensor(_CudaArray(hdst.data_ptr(), (N,), "|u1"), device="cuda")
hsrc = torch.ones(N, dtype=torch.uint8, pin_memory=True)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def run(ops):
    torch.cuda.synchronize()
    es = []
    for st, f in ops:
        a, b = ev(), ev()
        with torch.cuda.stream(st):
            a.record(); f(); b.record()
        es.append((a, b))
    torch.cuda.synchronize()
    return [round(N / a.elapsed_time(b) / 1e6, 2) for a, b in es]
G = lambda: t.gather(idx, out=gout)
CE_D2H = lambda: hdst.copy_(dsrc, non_blocking=True)
SM_D2H = lambda: torch.add(dsrc, 0, out=hview)
CE_H2D = lambda: gout.copy_(hsrc, non_blocking=True)
for name, ops in [("gather alone", [(s1, G)]), ("CE D2H alone", [(s2, CE_D2H)]), ("SM D2H alone", [(s2, SM_D2H)]),
                  ("gather + CE D2H", [(s1, G), (s2, CE_D2H)]), ("gather + SM D2H", [(s1, G), (s2, SM_D2H)]),
                  ("CE H2D + CE D2H", [(s1, CE_H2D), (s2, CE_D2H)]), ("CE H2D + SM D2H", [(s1, CE_H2D), (s2, SM_D2H)])]:
    run(ops)
    print(json.dumps({"case": name, "gbs_each": run(ops)}), flush=True)
