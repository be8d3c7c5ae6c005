"""Summarise an ncu report (and optionally a launch-list CSV) into a short text for profiles/.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep [--launches gpurun_out/launches.csv]
    python scripts/ncu_summary.py --traffic gpurun_out/traffic.csv --bench gpurun_out/t.json \
        [--out profiles/ncu_traffic.json]

The --traffic form reads a per-launch metrics CSV of the gather kernels inside bench.py's NVTX
"timed" range (ncu --nvtx --nvtx-include "timed/" --metrics dram__bytes_read.sum,...) and the
JSON line the same command printed, and records per-launch averages under the workload's name:
HBM bytes (dram read + write: roofline.traffic), link-side bytes (sysmem read sectors x 32) and
the algorithmic bytes (rows per step x rb).
"""
import argparse
import csv
import io
import json
import re
import os
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


def traffic(csv_path, bench_path, out_path):
    text = open(csv_path).read()
    rows = list(csv.reader(io.StringIO(text[text.index('"ID"'):])))
    h = rows[0]
    per = defaultdict(dict)
    for r in rows[1:]:
        name = r[h.index("Kernel Name")]
        if not re.search(r"\bk_(single|multi|narrow|runs|paper|bulk|share)\b", name):
            continue
        unit = r[h.index("Metric Unit")]
        v = float(r[h.index("Metric Value")].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3,
                 "ms": 1e6, "sector": 1, "request": 1}.get(unit, 1)
        per[r[h.index("ID")]][r[h.index("Metric Name")]] = v * scale
        per[r[h.index("ID")]]["kernel"] = name
    launches = list(per.values())
    n = len(launches)
    avg = lambda k: sum(x.get(k, 0.0) for x in launches) / max(1, n)
    line = json.loads([x for x in open(bench_path).read().splitlines() if x.startswith("{")][-1])
    cfg = line["config"]
    rec = {
        "plan": line["plan"], "table_memory": (line.get("table_memory") or "").split(" ")[0] or None,
        "launches": n,
        "kernel": launches[0]["kernel"] if n else None,
        "hbm_bytes_per_launch": round(avg("dram__bytes_read.sum") + avg("dram__bytes_write.sum")),
        "hbm_read_bytes_per_launch": round(avg("dram__bytes_read.sum")),
        "hbm_write_bytes_per_launch": round(avg("dram__bytes_write.sum")),
        "sysmem_bytes_per_launch": round(32 * avg("syslts__t_sectors_aperture_sysmem_op_read.sum")),
        "sysmem_requests_per_launch": round(avg("syslts__t_requests_aperture_sysmem_op_read.sum")),
        "pcie_read_bytes_per_launch": round(avg("pcie__read_bytes.sum")),
        "pcie_write_bytes_per_launch": round(avg("pcie__write_bytes.sum")),
        "ncu_ns_per_launch": round(avg("gpu__time_duration.sum")),
        "algorithmic_bytes_per_launch": round(cfg["rows_per_step_per_gpu"] * cfg["row_bytes"]),
        "source": f"ncu per-launch metrics of the gather kernels in bench.py's NVTX 'timed' range "
                  f"({os.path.basename(csv_path)}); algorithmic = rows per step x rb",
    }
    db = {}
    if os.path.exists(out_path):
        db = json.load(open(out_path))
    db[cfg["workload"]] = rec
    with open(out_path, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)
        f.write("\n")
    print(json.dumps({cfg["workload"]: rec}))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep", nargs="?")
    ap.add_argument("--launches")
    ap.add_argument("--traffic")
    ap.add_argument("--bench")
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                  "profiles", "ncu_traffic.json"))
    a = ap.parse_args()
    if a.traffic:
        return traffic(a.traffic, a.bench, a.out)
    h, u, vals = raw(a.rep) if a.rep else ([], [], [])
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
