"""NEXT-1 ablation: the paper's kernels (PyD Naive, PyD Optimized = circular shift) vs this
repo's kernel family on B200, over the paper's Fig. 8 widths (2048..2076 B, step 4)
and a Fig. 7-style grid. Random indices into a 4,194,304-row pool (reading: SURVEY c13).

Prints JSON lines: GB/s per (width, kernel) and, with --predict, the (warp, 128-B line) request
count the paper's model predicts for that kernel and index list (numpy form of
oracle/access_model.count_requests, computed here for large n)."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np


def predicted_requests(idx: np.ndarray, W: int, shift: bool, warp=32, L=32) -> int:
    """Distinct (warp, line) pairs of the thread-per-element kernel (4-B elements, 128-B lines,
    table base line-aligned) — the paper's request accounting (reading R14)."""
    n = idx.size
    r = np.repeat(np.arange(n, dtype=np.int64), W)
    j = np.tile(np.arange(W, dtype=np.int64), n)
    g = idx[r]
    if shift:
        s = ((r * W) - (g * W)) % L
        e = (j + s) % W
    else:
        e = j
    t = r * W + j
    key = (t // warp) * (1 << 40) + (g * W + e) // L
    return int(np.unique(key).size)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--widths", default="2048,2052,2056,2060,2064,2068,2072,2076")
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--pool", type=int, default=4194304)
    ap.add_argument("--predict", action="store_true")
    ap.add_argument("--once", action="store_true", help="one launch per kernel (for ncu)")
    args = ap.parse_args()
    import torch

    import paper_2101_07956_b200 as ut
    import workloads
    widths = [int(w) for w in args.widths.split(",")]
    tbytes = args.pool * max(widths)
    hb = workloads.HostBuffer(tbytes)
    workloads.fill_table(hb.addr, tbytes // 4096, 4096, 1, threads=0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for rb in widths:
        idx = workloads.uniform_idx(args.n, args.pool, seed=rb)
        idx_d = torch.from_numpy(idx).cuda()
        out = torch.empty(args.n * rb, dtype=torch.uint8, device="cuda")
        ref = None
        with ut.Table(hb.addr, args.pool, rb) as t:
            for name, plans in [("paper_naive", ["paper_naive"]), ("paper_shift", ["paper_shift"]),
                                ("ours_noreorder", ["auto", "reorder=off"]),
                                ("ours", ["auto", "reorder=auto"])]:
                for p in plans:
                    t.set_plan(p)
                ts = []
                for rep in range(1 if args.once else 5):
                    flush.zero_()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    t.gather(idx_d, out=out)
                    e1.record()
                    torch.cuda.synchronize()
                    ts.append(e0.elapsed_time(e1))
                got = out.cpu().numpy().tobytes()
                ref = ref or got
                rec = {"rb": rb, "kernel": name, "plan": t.plan, "n": args.n,
                       "gbs": round(args.n * rb / np.median(ts) / 1e6, 2), "same_bytes": got == ref}
                if args.predict and name.startswith("paper"):
                    rec["predicted_requests"] = predicted_requests(idx, rb // 4, name == "paper_shift")
                if args.predict and name.startswith("ours"):
                    a = (idx * rb) // 128
                    b = (idx * rb + rb - 1) // 128
                    rec["predicted_requests"] = int((b - a + 1).sum())   # lines touched per row
                print(json.dumps(rec), flush=True)
    hb.close()


if __name__ == "__main__":
    main()
