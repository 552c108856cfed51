"""Excess shared-memory wavefronts (bank conflicts) per CUDA source line from
`ncu -i REP --page source --csv --print-source cuda,sass --kernel-name K --launch-count 1`.
    python tools/ncu_smem_conflicts.py src.csv [N]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
hdr = next(r for r in rows if r and r[0] == "Line No")
ix, iw = hdr.index("L1 Wavefronts Shared Excessive"), hdr.index("L1 Wavefronts Shared")
per, tot, text = collections.Counter(), collections.Counter(), {}
cur, fname = None, ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) <= ix or r[0] == "Line No":
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        text[cur] = r[1]
    try:
        per[cur] += float(r[ix] or 0)
        tot[cur] += float(r[iw] or 0)
    except ValueError:
        pass
s = sum(per.values()) or 1.0
for ln, v in per.most_common(n):
    print(f"{100 * v / s:5.1f}%  excess {int(v):>9} of {int(tot[ln]):>9}  {ln[0]}:{ln[1]}: {text.get(ln, '').strip()[:90]}")
