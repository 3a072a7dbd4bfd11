#!/usr/bin/env python
"""Per-source-line SASS instruction counts (and local-memory LDL/STL) of one kernel.

    nvdisasm -g -c X.cubin > X.sass ; python tools/sass_lines.py X.sass FUNC_SUBSTR [FILE_SUBSTR]
"""
import re
import sys
from collections import defaultdict

path, fn = sys.argv[1], sys.argv[2]
fsub = sys.argv[3] if len(sys.argv) > 3 else ""
cur = None
infn = False
cnt = defaultdict(int)
loc = defaultdict(int)
for line in open(path):
    st = line.strip()
    if st.startswith(".text.") or ((st.startswith("$_Z") or st.startswith("_Z")) and st.endswith(":")):
        infn = fn in st.split("$")[-1]
        continue
    if not infn:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    if re.search(r"/\*[0-9a-f]{4,}\*/", line) and cur:
        cnt[cur] += 1
        if re.search(r"\b(LDL|STL)\b", line):
            loc[cur] += 1
tot = sum(cnt.values())
print(f"total SASS {tot}, local ld/st {sum(loc.values())}")
for k in sorted(cnt):
    if fsub in k[0] and (loc[k] or cnt[k] >= 1):
        print(f"{k[0]}:{k[1]:5d} {cnt[k]:6d} {'LOCAL ' + str(loc[k]) if loc[k] else ''}")
