"""Summarise an ncu report (and optionally a launch-list CSV) into a short text for profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv]
"""
import argparse
import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "syslts__t_sectors_srcunit_tex_aperture_sysmem_op_read_lookup_miss.sum",
    "syslts__t_requests_aperture_sysmem_op_read.sum",
    "syslts__t_sectors_aperture_sysmem_op_read.sum",
    "syslts__d_sectors_fill_sysmem.sum",
    "pcie__read_bytes.sum", "pcie__write_bytes.sum",
    "pcie__read_bytes.sum.per_second", "pcie__write_bytes.sum.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_requests_srcunit_tex_op_write.sum",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out[out.index('"ID"'):])))
    return rows[0], rows[1], rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--launches")
    a = ap.parse_args()
    h, u, vals = raw(a.rep)
    for v in vals:
        name = v[h.index("Kernel Name")]
        print(f"kernel: {name}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"  {k:75s} {v[i]:>18s} {u[i]}")
        stalls = [(float(v[i]), k) for i, k in enumerate(h)
                  if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")
                  and v[i] not in ("", "n/a")]
        stalls.sort(reverse=True)
        tot = sum(s for s, _ in stalls) or 1.0
        print("  top stall reasons (pc sampling share):")
        for s, k in stalls[:5]:
            print(f"    {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):40s} {100 * s / tot:5.1f} %")
    if a.launches:
        text = open(a.launches).read()
        rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
        hh = rows[0]
        agg = defaultdict(lambda: [0, 0.0])
        for r in rows[1:]:
            if r[hh.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            k = r[hh.index("Kernel Name")]
            agg[k][0] += 1
            agg[k][1] += float(r[hh.index("Metric Value")])
        tot = sum(t for _, t in agg.values()) or 1.0
        print("launch list (ncu gpu__time_duration.sum, cold-cache, serialised):")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            print(f"  {100 * t / tot:5.1f} %  {n:4d} launches  {t / n / 1e3:10.1f} us/launch  {k[:90]}")


if __name__ == "__main__":
    sys.exit(main())
