"""Experiment: host->host e2e (ut_gather_host, direct stores into mapped pinned output) vs row
width on a 1-GiB table with uniform indices: do partial-line writes (rows not a multiple of
128 B) cost link capacity beyond their bytes? Prints kernel-to-HBM GB/s and e2e GB/s per rb."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_07956_b200 as ut
import workloads


def main():
    for rb in [int(x) for x in (sys.argv[1:] or "256 384 400 512 1024 2048 2408".split())]:
        rows = (1 << 30) // rb
        n = (192 << 20) // rb
        hb = workloads.HostBuffer(rows * rb)
        workloads.fill_table(hb.addr, rows, rb, 5, threads=16)
        t = ut.Table(hb.addr, rows, rb)
        t.set_plan("stage=" + os.environ.get("UT_E2E_STAGE", "auto"))
        idx_h = [torch.from_numpy(workloads.uniform_idx(n, rows, s)).pin_memory() for s in range(4)]
        out_h = torch.empty(n * rb, dtype=torch.uint8, pin_memory=True)
        out_d = torch.empty(n * rb, dtype=torch.uint8, device="cuda")
        idx_d = [x.cuda() for x in idx_h]

        def timed(fn):
            fn(0); torch.cuda.synchronize()
            sec = 0.0
            for s in range(1, 4):
                torch.cuda.synchronize(); t0 = time.perf_counter()
                fn(s); torch.cuda.synchronize()
                sec += time.perf_counter() - t0
            return round(3 * n * rb / sec / 1e9, 2)

        k = timed(lambda s: t.gather(idx_d[s], out=out_d))
        e = timed(lambda s: t.gather_host(idx_h[s], out_host=out_h))
        print(json.dumps({"rb": rb, "rb_mod_128": rb % 128, "to_hbm_gbs": k, "e2e_direct_gbs": e,
                          "stage": os.environ.get("UT_E2E_STAGE", "auto")}), flush=True)
        t.close(); hb.close()


if __name__ == "__main__":
    main()
