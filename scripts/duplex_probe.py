"""Experiment: host-link duplex behaviour (dev aid). Bidirectional memcpy, gather under D2H load,
and ut_gather_host chunk sizes."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2101_07956_b200 as ut
import workloads


def ev():
    return torch.cuda.Event(enable_timing=True)


def main():
    N = 1 << 30
    hA = torch.empty(N, dtype=torch.uint8, pin_memory=True); hA.fill_(1)
    hB = torch.empty(N, dtype=torch.uint8, pin_memory=True)
    dA = torch.empty(N, dtype=torch.uint8, device="cuda")
    dB = torch.empty(N, dtype=torch.uint8, device="cuda"); dB.fill_(2)
    sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(sA):
            dA.copy_(hA, non_blocking=True)
        with torch.cuda.stream(sB):
            hB.copy_(dB, non_blocking=True)
        torch.cuda.synchronize()
        el = time.perf_counter() - t0
    print(json.dumps({"bidir_memcpy_total_gbs": round(2 * N / el / 1e9, 2), "s": round(el, 4)}), flush=True)
    # gather alone vs gather with a concurrent D2H stream
    rows, rb = (1 << 30) // 512, 512
    hb = workloads.HostBuffer(rows * rb)
    workloads.fill_table(hb.addr, rows, rb, 1)
    idx = torch.from_numpy(workloads.uniform_idx(1 << 20, rows, 3)).cuda()
    out = torch.empty((1 << 20) * rb, dtype=torch.uint8, device="cuda")
    t = ut.Table(hb.addr, rows, rb)
    for mode in ["alone", "with_d2h", "with_h2d"]:
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        if mode == "with_d2h":
            with torch.cuda.stream(sB):
                hB.copy_(dB, non_blocking=True)
        if mode == "with_h2d":
            with torch.cuda.stream(sB):
                dA.copy_(hA, non_blocking=True)
        e0.record()
        t.gather(idx, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(json.dumps({"gather_512B": mode, "gbs": round(out.numel() / ms / 1e6, 2)}), flush=True)
    t.close()
    hb.close()


if __name__ == "__main__":
    if len(sys.argv) > 1:
        main()
    else:
        main()
        for chunk in [1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20]:
            env = dict(os.environ, UT_HOST_CHUNK=str(chunk))
            p = subprocess.run([sys.executable, "bench.py", "--config", "products", "--steps", "20",
                                "--no-cpu"], capture_output=True, text=True, env=env)
            for l in p.stdout.splitlines():
                if l.startswith("{"):
                    d = json.loads(l)
                    print(json.dumps({"chunk": chunk, "e2e": d["e2e"]["value"], "value": d["value"]}), flush=True)
