"""Top SASS instructions by warp-stall samples from `ncu -i REP --page source
--csv [--kernel-name K --launch-count 1]` output (per-instruction view).

    python tools/ncu_hot.py src.csv [N]
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
hdr = rows[1]
ia, isrc, ist = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    if len(r) <= ist:
        continue
    try:
        data.append((float(r[ist] or 0), r[ia], r[isrc]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1.0
for v, addr, src in sorted(data, reverse=True)[:n]:
    print(f"{100 * v / tot:5.1f}%  {addr}  {src[:120]}")
