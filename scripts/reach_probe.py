"""Experiment: how much index locality does the translation path need? (development aid)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2101_07956_b200 as ut
import workloads
from xlat_probe import tgather


def main():
    tbytes = 16 << 30
    hb = workloads.HostBuffer(tbytes)
    workloads.fill_table(hb.array(), tbytes // 4096, 4096, 1)
    n = 1 << 20
    for gib in [1, 1.5, 2, 3]:
        for rb in [64, 512]:
            rows = int(gib * (1 << 30)) // rb
            idx = workloads.uniform_idx(n, rows, seed=rb)
            with ut.Table(hb.addr, rows, rb) as t:
                ms = tgather(t, torch.from_numpy(idx).cuda(), torch.empty(n * rb, dtype=torch.uint8, device="cuda"))
            print(json.dumps({"gib": gib, "rb": rb, "order": "random", "gbs": round(n * rb / ms / 1e6, 2),
                              "mrows_s": round(n / ms / 1e3, 1)}), flush=True)
    rng = np.random.default_rng(0)
    for rb in [64, 512]:
        rows = tbytes // rb
        idx = workloads.uniform_idx(n, rows, seed=rb)
        out = torch.empty(n * rb, dtype=torch.uint8, device="cuda")
        orders = {"random": idx, "sorted": np.sort(idx)}
        for k in [21, 24, 26, 27, 28, 29, 30, 31]:
            b = (idx * rb) >> k
            orders[f"bucket{k}"] = idx[np.argsort(b, kind="stable")]
        b = (idx * rb) >> 21
        ub = np.unique(b)
        perm = rng.permutation(ub.size)
        key = perm[np.searchsorted(ub, b)]
        orders["bucket21_shuffled"] = idx[np.argsort(key, kind="stable")]
        b = (idx * rb) >> 26
        ub = np.unique(b)
        perm = rng.permutation(ub.size)
        key = perm[np.searchsorted(ub, b)]
        orders["bucket26_shuffled"] = idx[np.argsort(key, kind="stable")]
        with ut.Table(hb.addr, rows, rb) as t:
            for name, o in orders.items():
                ms = tgather(t, torch.from_numpy(np.ascontiguousarray(o)).cuda(), out)
                print(json.dumps({"gib": 16, "rb": rb, "order": name, "gbs": round(n * rb / ms / 1e6, 2),
                                  "mrows_s": round(n / ms / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
