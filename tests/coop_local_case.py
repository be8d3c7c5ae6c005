"""Helper of tests/test_round2_gpu.py::test_coop_in_process_ranks (run as its own process):
`world` in-process ranks of the cooperative gather on device 0 over one managed table, each
rank's rows checked against the oracle, and the owners' host rows per step against the union of
the ranks' valid ids. Prints COOP-LOCAL-OK on success."""
import os
import sys
import threading

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import paper_2101_07956_b200 as ut  # noqa: E402
import workloads  # noqa: E402


def main(world: int) -> None:
    rows, rb = 60_000, 400
    torch.cuda.set_device(0)
    with ut.Table.create(rows, rb, "managed") as t:
        workloads.fill_table(t.host_addr, rows, rb, 701)
        lists = [workloads.uniform_idx(20_000 + 13 * r, rows // 4, 710 + r) for r in range(world)]
        lists[0][5] = rows + 2                       # one out-of-range id on rank 0
        wants = [oracle.gather(t.host_addr, rows, rb, l) for l in lists]
        max_n = max(l.size for l in lists)
        coops = [ut.Coop(t, max_n, rank=r, world=world, sync="device", local=True)
                 for r in range(world)]
        for c in coops:
            c.open_local(coops)
        idx = [torch.from_numpy(l).cuda() for l in lists]
        streams = [torch.cuda.Stream() for _ in range(world)]
        outs = [torch.empty(l.size * rb, dtype=torch.uint8, device="cuda") for l in lists]
        torch.cuda.synchronize()
        errs = []

        def step(r):
            try:
                torch.cuda.set_device(0)
                for _ in range(3):                   # several steps: parity double-buffering
                    coops[r].gather(idx[r], out=outs[r], stream=streams[r])
                streams[r].synchronize()
            except Exception as e:   # pragma: no cover
                errs.append(repr(e))

        th = [threading.Thread(target=step, args=(r,)) for r in range(world)]
        [x.start() for x in th]
        [x.join() for x in th]
        assert not errs, errs
        for r in range(world):
            assert outs[r].cpu().numpy().tobytes() == wants[r][0].tobytes(), r
            assert coops[r].error_pos(streams[r]) == wants[r][1], r
        valid = np.concatenate([l[(l >= 0) & (l < rows)] for l in lists])
        fetched = sum(c.stats()["last_unique_rows"] for c in coops)
        assert fetched == np.unique(valid).size, (fetched, np.unique(valid).size)
        for c in coops:
            c.close()
    print("COOP-LOCAL-OK", world)


if __name__ == "__main__":
    main(int(sys.argv[1]))
