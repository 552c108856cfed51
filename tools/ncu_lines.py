"""Warp-stall samples per CUDA source line from
`ncu -i REP --page source --csv --kernel-name K --launch-count 1 --print-source cuda,sass`.

    python tools/ncu_lines.py src.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 15
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ist = hdr.index("Warp Stall Sampling (All Samples)")
per = collections.Counter()
text = {}
cur = None
fname = ""
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) <= ist or (r and r[0] == "Line No"):
        continue
    if r[0]:
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        text[cur] = r[1]
    try:
        per[cur] += float(r[ist] or 0)
    except ValueError:
        pass
tot = sum(per.values()) or 1.0
for ln, v in per.most_common(n):
    print(f"{100 * v / tot:5.1f}%  {ln[0]}:{ln[1]}: {text.get(ln, '').strip()[:100]}")
