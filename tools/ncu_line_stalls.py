"""Warp-stall samples per CUDA source line of one ncu capture (the source page
with --print-source cuda,sass): where a kernel's warps wait, and on what.

    ncu -i REP --page source --csv --print-source cuda,sass --launch-count 1 > src.csv
    python tools/ncu_line_stalls.py src.csv [N]
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = next(r for r in rows if r and r[0] == "Line No")
i_all = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [(i, h[len("stall_"):]) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
per = collections.Counter()
why = collections.defaultdict(collections.Counter)
text = {}
cur, fname = None, ""
for r in rows:
    if r and r[0] == "File Name":
        fname = r[1].rsplit("/", 1)[-1]
        continue
    if len(r) <= i_all or r[0] == "Line No":
        continue
    if r[0]:   # a CUDA source line (SASS rows that follow have an empty first column)
        try:
            cur = (fname, int(r[0]))
        except ValueError:
            continue
        text[cur] = r[1]

    def f(x):
        try:
            return float(x or 0)
        except ValueError:
            return 0.0
    if not r[0]:
        per[cur] += f(r[i_all])
        for i, nm in stall_cols:
            why[cur][nm] += f(r[i])
tot = sum(per.values()) or 1.0
print(f"{int(tot)} samples")
for ln, v in per.most_common(n):
    top = ", ".join(f"{k} {100 * c / v:.0f}%" for k, c in why[ln].most_common(2) if c)
    print(f"{100 * v / tot:5.1f}%  {ln[0]}:{ln[1]:<5} {text.get(ln, '').strip()[:70]:70s} [{top}]")
