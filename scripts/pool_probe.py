"""Cost of a unified tensor's allocation with and without the recycling pool.

For each kind and size: the mean wall time of one create + release of a table through ut_create
(one backend allocation + free per tensor) and through ut_pool_table (a cached block after the
first), and of a bare ut_pool_alloc/free pair. One JSON line per case."""
import json
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2101_07956_b200 as ut  # noqa: E402


def per_call(fn, n):
    fn()                                           # warm: the pool's first block, CUDA context
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    torch.cuda.init()
    torch.empty(1, device="cuda")
    for kind in ("pinned", "managed"):
        for nbytes in (4096, 1 << 20, 64 << 20, 512 << 20):
            rows, rb = nbytes // 512, 512
            n = 200 if nbytes <= (1 << 20) else (20 if nbytes <= (64 << 20) else 5)
            pool = ut.Pool(kind)

            def plain():
                h, _ = ut.ut_create(0, rows, rb, ut.UT_ALLOC[kind])
                ut.ut_release(h)

            def pooled():
                h, _ = ut.ut_pool_table(pool.handle, 0, rows, rb)
                ut.ut_release(h)

            def block():
                a, _ = pool.alloc(nbytes)
                pool.free(a)

            row = {"kind": kind, "bytes": nbytes, "iters": n,
                   "create_release_us": round(per_call(plain, n), 2),
                   "pool_table_release_us": round(per_call(pooled, n), 2),
                   "pool_alloc_free_us": round(per_call(block, n), 3)}
            row["speedup"] = round(row["create_release_us"] / row["pool_table_release_us"], 1)
            row["pool"] = pool.stats()
            print(json.dumps(row), flush=True)
            pool.release_cached()
            pool.close()


if __name__ == "__main__":
    main()
