"""Per-sweep kernel times of the last CNN round in an ncu launch-list CSV
(gpu__time_duration.sum): which kernels cost what in the head / tail sweeps.

    python tools/sweep_profile.py gpurun_out/launches.csv
"""
import collections
import csv
import re
import sys

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
seq = []
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    name = re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1].split("<")[0].replace("void ", "")
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    ms = v / 1e6 if unit == "ns" else v / 1e3 if unit == "us" else v
    seq.append((name, ms, r["Grid Size"]))
# sweeps start at k_fwd (k_slots before it at a low-rank switch step, and in
# captures older than the slots-in-k_fwd change); keep the last round (the
# last run of consecutive sweeps)
starts = []
for i, (n, _, _) in enumerate(seq):
    if n == "k_slots" or (n == "k_fwd" and not (i > 0 and seq[i - 1][0] == "k_slots")):
        starts.append(i)
rounds, cur = [], [starts[0]]
for a, b in zip(starts, starts[1:]):
    gap = any(not seq[j][0].startswith("k_") for j in range(a, b))
    if gap:
        rounds.append(cur)
        cur = [b]
    else:
        cur.append(b)
rounds.append(cur)
last = rounds[-1]
print(f"{len(rounds)} rounds; last has {len(last)} sweeps")
bounds = last + [last[-1] + 1 + next((k for k, (n, _, _) in enumerate(seq[last[-1] + 1:]) if not n.startswith("k_")), 0)]
per = collections.OrderedDict()
tot = collections.Counter()
for si, (a, b) in enumerate(zip(bounds, bounds[1:])):
    row = collections.Counter()
    for n, ms, g in seq[a:b]:
        row[n] += ms
        tot[n] += ms
    per[si] = row
names = [n for n, _ in tot.most_common()]
print("kernel totals (ms):", {n: round(tot[n], 2) for n in names}, "sum", round(sum(tot.values()), 2))
print("sweep " + " ".join(f"{n[:10]:>10}" for n in names))
for si, row in per.items():
    if si < 6 or si % 8 == 0 or si > len(per) - 3:
        print(f"{si:5d} " + " ".join(f"{row[n]:10.3f}" for n in names))
# head (first 24) vs tail
for lo, hi in ((0, 24), (24, len(per))):
    c = collections.Counter()
    for si in range(lo, hi):
        c.update(per[si])
    print(f"sweeps {lo}-{hi}: " + ", ".join(f"{n} {c[n]:.2f}" for n in names))
