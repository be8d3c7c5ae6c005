"""Experiment: where does e2e.to_hbm (pinned idx H2D + gather into HBM + 8-B read-back) lose time
against the device-timed gather on the reddit shape? Variants timed on the host, per step."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2101_07956_b200 as ut
import workloads


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "reddit"
    spec = bench.workload_spec(cfg)
    rows, rb = spec["rows"], spec["row_bytes"]
    lists = bench.make_index_lists(spec, 0, 1, 12, 2118, 8)
    hb = workloads.HostBuffer(rows * rb); workloads.fill_table(hb.addr, rows, rb, 2101, threads=16)
    t = ut.Table(hb.addr, rows, rb)
    max_n = max(l.size for l in lists)
    out = torch.empty(max_n * rb, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    idx_h = [torch.from_numpy(l).pin_memory() for l in lists]
    idx_d = [x.cuda() for x in idx_h]
    probe = torch.empty(1, dtype=torch.int64, pin_memory=True)

    def run(name, step, do_flush=True):
        for s in range(2):
            step(s)
        torch.cuda.synchronize()
        sec, nb = 0.0, 0
        for s in range(2, len(lists)):
            if do_flush:
                flush.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            step(s)
            torch.cuda.synchronize()
            sec += time.perf_counter() - t0
            nb += lists[s].size * rb
        print(json.dumps({"cfg": cfg, "case": name, "flush": do_flush, "gbs": round(nb / sec / 1e9, 2)}), flush=True)

    def g_dev(s):
        t.gather(idx_d[s], out=out[: lists[s].size * rb])

    def g_h2d(s):
        d = idx_h[s].to("cuda", non_blocking=True)
        t.gather(d, out=out[: lists[s].size * rb])

    def g_full(s):
        d = idx_h[s].to("cuda", non_blocking=True)
        r = t.gather(d, out=out[: lists[s].size * rb])
        probe.copy_(r[:8].view(torch.int64), non_blocking=False)

    for fl in (True, False):
        run("gather, idx resident", g_dev, fl)
        run("idx H2D + gather", g_h2d, fl)
        run("idx H2D + gather + 8-B read-back", g_full, fl)
    out_h = torch.empty(max_n * rb, dtype=torch.uint8, pin_memory=True)
    run("ut_gather_host direct (host -> host)", lambda s: t.gather_host(idx_h[s], out_host=out_h))
    run("idx H2D + gather + 8-B read-back, after gather_host", g_full)
    run("gather, idx resident, after gather_host", g_dev)
    del out_h
    run("gather, idx resident, pinned output freed", g_dev)


if __name__ == "__main__":
    main()
