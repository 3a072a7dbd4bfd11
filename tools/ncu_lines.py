#!/usr/bin/env python
"""ncu stall samples of one kernel per CUDA source line: join the SASS source page of an
ncu report (function-relative addresses) with nvdisasm's line table of the same binary.

    ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv
    cuobjdump -xelf all libgls.so; nvdisasm -g -c gls_kernels.sm_100a.cubin > k.sass
    python tools/ncu_lines.py X.csv k.sass FUNC_SUBSTR [N]
"""
import csv
import re
import sys
from collections import defaultdict

csvp, sassp, fn = sys.argv[1], sys.argv[2], sys.argv[3]
N = int(sys.argv[4]) if len(sys.argv) > 4 else 40
# address -> (file, line), innermost inlined location
line_of = {}
cur, infn = None, False
for line in open(sassp):
    st = line.strip()
    if st.startswith(".text.") or ((st.startswith("$_Z") or st.startswith("_Z")) and st.endswith(":")):
        if st.startswith(".text.") or not st.startswith("$"):
            infn = fn in st
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/", line)
    if m and cur:
        line_of[int(m.group(1), 16)] = cur
rows = list(csv.reader(open(csvp)))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
ia, iex = h.index("Address"), h.index("Instructions Executed")
ith = h.index("Thread Instructions Executed")
iall = h.index("Warp Stall Sampling (All Samples)")
f = lambda x: float(x.replace(",", "") or 0)
base = None
agg = defaultdict(lambda: defaultdict(float))
for r in rows[hdr + 1:]:
    if len(r) <= ith or not r[ia].startswith("0x"):
        continue
    a = int(r[ia], 16)
    base = a if base is None else base
    off = a - base
    key = line_of.get(off, ("?", 0))
    d = agg[key]
    d["samples"] += f(r[iall])
    d["inst"] += f(r[iex])
    d["thr"] += f(r[ith])
    for c in cols:
        d[c] += f(r[h.index(c)])
tot = sum(d["samples"] for d in agg.values())
toti = sum(d["inst"] for d in agg.values())
print(f"samples {tot:.0f}, warp instructions {toti:.4g}, lines {len(agg)}, mapped addresses {len(line_of)}")
for k, d in sorted(agg.items(), key=lambda x: -x[1]["samples"])[:N]:
    top = sorted(((d[c], c[6:]) for c in cols), reverse=True)[:3]
    print(f"{k[0]}:{k[1]:<5d} {d['samples'] / tot:6.1%} inst {d['inst'] / toti:6.1%} thr "
          f"{d['thr'] / max(1, d['inst']):5.1f}  " + " ".join(f"{n} {v / max(1, d['samples']):.0%}" for v, n in top))
# ranges of gls_lanes.cuh lines given as LO-HI arguments after N: samples and stall mix per range
for rg in sys.argv[5:]:
    lo, hi = (int(x) for x in rg.split("-"))
    sel = [d for k, d in agg.items() if k[0] == "gls_lanes.cuh" and lo <= k[1] <= hi]
    s = sum(d["samples"] for d in sel)
    ins = sum(d["inst"] for d in sel)
    th = sum(d["thr"] for d in sel)
    mix = sorted(((sum(d[c] for d in sel), c[6:]) for c in cols), reverse=True)[:6]
    print(f"lines {lo}-{hi}: samples {s / tot:.1%}, inst {ins / toti:.1%} ({ins:.3g}), thr {th / max(1, ins):.1f}: "
          + " ".join(f"{n} {v / max(1, s):.0%}" for v, n in mix))
