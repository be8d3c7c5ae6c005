"""User-level effect of the unified allocator's recycling: hybrid ops whose
Table 3 output is a unified tensor (a new allocation per op), timed with the storage taken from the
recycling pool and, for comparison, from a fresh ut_create per tensor. One JSON line per case."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2101_07956_b200 import unified as U  # noqa: E402


def rate(fn, n):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    torch.cuda.init()
    for shape in ((256, 64), (4096, 128), (65536, 128)):
        a = torch.randn(*shape)
        u = U.to_unified(a)                                      # propagated
        b = torch.randn(*shape)                                  # CPU operand: R1 -> unified out
        idx = torch.randint(0, shape[0], (shape[0] // 4,), device="cuda")
        v = U.to_unified(a, propagatedToCUDA=False)              # v[gpu idx] -> unified output

        def add():
            (u + b).close()

        def gather():
            v[idx].close()

        row = {"shape": list(shape)}
        for name, fn in (("add_cpu_operand", add), ("gather_unified_out", gather)):
            saved = U._POOLED
            n = 200 if shape[0] <= 4096 else 50
            row[name + "_pooled_us"] = round(rate(fn, n), 1)
            U._POOLED = ()                                       # every tensor a fresh ut_create
            row[name + "_fresh_us"] = round(rate(fn, n), 1)
            U._POOLED = saved
        row["allocator"] = U.allocator_stats("managed")
        print(json.dumps(row), flush=True)
        u.close()
        v.close()


if __name__ == "__main__":
    main()
