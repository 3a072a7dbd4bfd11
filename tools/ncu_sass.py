#!/usr/bin/env python
"""Aggregate ncu's SASS source page: executed instructions by opcode, the hottest
instructions (stall samples), and local-memory (LDL/STL) executions.

    ncu -i X.ncu-rep --page source --csv --print-source sass > X.csv; python tools/ncu_sass.py X.csv [N]
"""
import csv
import sys
from collections import defaultdict

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hdr]
ia, isrc, ismp, iex, ith = (h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)"),
                            h.index("Instructions Executed"), h.index("Thread Instructions Executed"))
ins = []
for r in rows[hdr + 1:]:
    if len(r) <= ith or not r[ia].startswith("0x"):
        continue
    f = lambda x: float(x.replace(",", "") or 0)
    ins.append((int(r[ia], 16), r[isrc].strip(), f(r[ismp]), f(r[iex]), f(r[ith])))
tot_ex = sum(x[3] for x in ins)
tot_th = sum(x[4] for x in ins)
tot_s = sum(x[2] for x in ins)
print(f"instructions executed {tot_ex:.4g}, threads/inst {tot_th / max(1, tot_ex):.2f}, samples {tot_s:.0f}")
op = defaultdict(float)
for a, s, smp, ex, th in ins:
    o = s.split()[0] if not s.startswith("@") else s.split()[1]
    op[o.split(".")[0]] += ex
print("by opcode:", ", ".join(f"{k} {v / tot_ex:.1%}" for k, v in sorted(op.items(), key=lambda x: -x[1])[:25]))
loc = [(ex, a, s) for a, s, smp, ex, th in ins if " LDL" in " " + s.replace("@", " ") or " STL" in " " + s.replace("@", " ")]
print(f"local ld/st executed {sum(x[0] for x in loc):.4g}")
base = ins[0][0] if ins else 0
for ex, a, s in sorted(loc, reverse=True)[:12]:
    print(f"  {ex:12.4g}  +{a - base:#x}  {s}")
print("hottest by stall samples:")
for a, s, smp, ex, th in sorted(ins, key=lambda x: -x[2])[:int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"  {smp / tot_s:6.2%} ex {ex:10.4g} thr {th / max(1, ex):5.1f}  +{a - base:#x}  {s}")
