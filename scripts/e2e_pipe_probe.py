"""Experiment: host->host e2e with the gather into HBM chunks on one stream and an SM copy-out
of finished chunks into mapped pinned host memory on a second stream (duplex probe: SM reads +
SM writes share the link better than SM reads + copy-engine writes). Prints e2e GB/s per chunk
size and copy-out grid."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2101_07956_b200 as ut
import workloads
from paper_2101_07956_b200.unified import _CudaArray

def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "products"
    spec = bench.workload_spec(cfg)
    rows, rb = spec["rows"], spec["row_bytes"]
    lists = bench.make_index_lists(spec, 0, 1, 8, 2118, 8)
    hb = workloads.HostBuffer(rows * rb); workloads.fill_table(hb.addr, rows, rb, 2101, threads=16)
    t = ut.Table(hb.addr, rows, rb)
    max_n = max(l.size for l in lists)
    idx_h = [torch.from_numpy(l).pin_memory() for l in lists]
    out_h = torch.empty(max_n * rb, dtype=torch.uint8, pin_memory=True)
    hview = torch.as_tensor(_CudaArray(out_h.data_ptr(), (max_n * rb,), "|u1"), device="cuda")
    idx_d = torch.empty(max_n, dtype=torch.int64, device="cuda")
    s1, s2 = torch.cuda.current_stream(), torch.cuda.Stream()

    def direct(ih):
        t.gather_host(ih, out_host=out_h)

    def pipe(ih, chunk_rows, nbuf=3):
        n = ih.numel()
        idx_d[:n].copy_(ih, non_blocking=True)
        bufs = [torch.empty(chunk_rows * rb, dtype=torch.uint8, device="cuda") for _ in range(nbuf)]
        done = [None] * nbuf
        k = 0
        for off in range(0, n, chunk_rows):
            c = min(chunk_rows, n - off)
            b = k % nbuf
            if done[b] is not None:
                s1.wait_event(done[b])
            t.gather(idx_d[off:off + c], out=bufs[b][: c * rb], stream=s1)
            ev = torch.cuda.Event(); ev.record(s1)
            s2.wait_event(ev)
            with torch.cuda.stream(s2):
                hview[off * rb:(off + c) * rb].copy_(bufs[b][: c * rb])
                d = torch.cuda.Event(); d.record(s2)
            done[b] = d
            k += 1
        s2.synchronize(); s1.synchronize()

    def rate(fn, *a):
        fn(idx_h[0], *a); torch.cuda.synchronize()
        sec, nb = 0.0, 0
        for ih in idx_h[1:]:
            torch.cuda.synchronize(); t0 = time.perf_counter()
            fn(ih, *a)
            torch.cuda.synchronize(); sec += time.perf_counter() - t0; nb += ih.numel() * rb
        return round(nb / sec / 1e9, 2)

    print(json.dumps({"cfg": cfg, "path": "direct-first", "e2e": rate(direct)}), flush=True)
    # parity of the pipe path
    pipe(idx_h[0], 16384)
    want, _ = __import__("oracle").gather(hb.addr, rows, rb, lists[0])
    assert out_h[: lists[0].size * rb].numpy().tobytes() == want.tobytes()
    print(json.dumps({"cfg": cfg, "path": "direct", "e2e": rate(direct)}), flush=True)
    print(json.dumps({"cfg": cfg, "path": "direct-again", "e2e": rate(direct)}), flush=True)
    for cr in (4096, 16384, 65536):
        print(json.dumps({"cfg": cfg, "path": "pipe-smcopy", "chunk_rows": cr, "e2e": rate(pipe, cr)}), flush=True)


if __name__ == "__main__":
    main()
