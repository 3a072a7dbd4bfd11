#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) or a launch-list CSV into profiles/.

    python profiles/summarize.py report.ncu-rep  > profiles/<name>.txt
    python profiles/summarize.py launches.csv    > profiles/<name>.txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__sass_inst_executed_op_local_ld.sum", "smsp__sass_inst_executed_op_local_st.sum",
    "smsp__sass_inst_executed_op_global_ld.sum", "smsp__sass_inst_executed_op_global_st.sum",
]


def rep(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        print(f"kernel: {d.get('Kernel Name')}  grid {d.get('launch__grid_size')} x {d.get('launch__block_size')}")
        for k in KEYS:
            if k in d:
                print(f"  {k:60s} {d[k]:>20s} {u.get(k, '')}")
        st = []
        for k, v in d.items():
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued"):
                try:
                    st.append((float(v.replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1.0
        print("  warp stall samples (share):")
        for v, k in sorted(st, reverse=True)[:10]:
            print(f"    {k:32s} {100 * v / tot:6.1f} %")


def launches(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    tot = {}
    for r in rows[hdr + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            t = float(r[vi].replace(",", ""))
            n, s = tot.get(name, (0, 0.0))
            tot[name] = (n + 1, s + t)
    all_t = sum(s for _, s in tot.values()) or 1.0
    unit = h[h.index("Metric Unit")] if "Metric Unit" in h else ""
    print(f"{'kernel':50s} {'launches':>9s} {'total':>14s} {'share':>7s}   (durations in ncu's unit {unit})")
    for name, (n, s) in sorted(tot.items(), key=lambda x: -x[1][1]):
        print(f"{name[:50]:50s} {n:9d} {s:14.0f} {100 * s / all_t:6.1f} %")


if __name__ == "__main__":
    p = sys.argv[1]
    (rep if p.endswith(".ncu-rep") else launches)(p)
