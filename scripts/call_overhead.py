"""Host-side cost of one ut_gather call (small n: launch-bound) — dev aid."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2101_07956_b200 as ut, workloads
rows, rb = 1024, 68
hb = workloads.HostBuffer(rows * rb); workloads.fill_table(hb.addr, rows, rb, 1)
t = ut.Table(hb.addr, rows, rb)
idx = torch.from_numpy(workloads.uniform_idx(512, rows, 2)).cuda()
out = torch.empty(512 * rb, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for _ in range(100): ut.ut_gather(t.handle, idx.data_ptr(), 512, out.data_ptr(), st)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N): ut.ut_gather(t.handle, idx.data_ptr(), 512, out.data_ptr(), st)
host = (time.perf_counter() - t0) / N
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(N): ut.ut_gather(t.handle, idx.data_ptr(), 512, out.data_ptr(), st)
e1.record(); torch.cuda.synchronize()
print({"host_us_per_call": round(host * 1e6, 2), "device_us_per_call": round(e0.elapsed_time(e1) / N * 1e3, 2)})
