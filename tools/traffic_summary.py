"""DRAM traffic per kernel class over one bench round, from
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --csv`
(every launch of the round).  Writes profiles/<name>.json (read by bench.py
for the roofline `traffic` field) and prints a markdown table.

    python tools/traffic_summary.py gpurun_out/traffic.csv profiles/r1_traffic
"""
import collections
import csv
import json
import re
import sys

CLASS = [("k_head_tail", "cnn_head"), ("k_head", "cnn_head"), ("k_fwd", "cnn_fwd"),
         ("k_bwd_conv", "cnn_bwd_conv"), ("k_wgrad", "cnn_wgrad"), ("k_lz_xt", "cnn_lz_xt"),
         ("k_lz_gram<1>", "cnn_lz_gram_fwd"), ("k_lz_gram<0>", "cnn_lz_gram_bwd"),
         ("k_lz_gram<true>", "cnn_lz_gram_fwd"), ("k_lz_gram<false>", "cnn_lz_gram_bwd"),
         ("k_lz_fwd_epi", "cnn_lz_fwd"), ("k_lz_fwd", "cnn_lz_fwd"), ("k_lz_bwd", "cnn_lz_bwd"),
         ("k_lz_fold", "cnn_lz_mat"), ("k_lz_mat", "cnn_lz_mat"), ("k_slots", "cnn_slots")]

rows = list(csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")))
per = collections.defaultdict(dict)
for r in rows:
    key = (r["ID"], r["Kernel Name"])
    v = float(r["Metric Value"].replace(",", ""))
    unit = r["Metric Unit"]
    if r["Metric Name"].startswith("dram__bytes"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        per[key][r["Metric Name"]] = v * scale
    else:
        per[key]["ms"] = v / 1e6 if unit == "ns" else v / 1e3 if unit == "us" else v
tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
for (_, name), m in per.items():
    base = re.sub(r"\(.*", "", name).split("::")[-1].replace("void ", "").strip()
    if base.startswith("k_lz_gram"):   # template args may be printed as <(bool)1, (int)8>
        cls = "cnn_lz_gram_fwd" if re.search(r"k_lz_gram<(\(bool\))?(1|true)", name) else "cnn_lz_gram_bwd"
    else:
        cls = next((c for k, c in CLASS if base == k or base.startswith(k)), None)
    if cls is None:
        continue
    t = tot[cls]
    t[0] += 1
    t[1] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    t[2] += m.get("ms", 0.0)
out = {c: {"launches": n, "dram_bytes": b, "dram_bytes_per_launch": b / n, "ms": ms,
           "dram_gbs": b / (ms / 1e3) / 1e9 if ms else None} for c, (n, b, ms) in tot.items()}
meta = {"source": sys.argv[1], "what": "ncu dram__bytes_read.sum + dram__bytes_write.sum over every launch "
        "of one C2 bench round (tools/profile_round.py); cold, serialised launches"}
json.dump({"meta": meta, "kernels": out}, open(sys.argv[2] + ".json", "w"), indent=1)
print("| kernel class | launches | DRAM GB / round | MB / launch | ms / round (ncu) | DRAM GB/s |")
print("|---|---|---|---|---|---|")
for c, v in sorted(out.items(), key=lambda x: -x[1]["ms"]):
    print(f"| {c} | {v['launches']} | {v['dram_bytes'] / 1e9:.2f} | {v['dram_bytes_per_launch'] / 1e6:.1f} | "
          f"{v['ms']:.2f} | {v['dram_gbs'] or 0:.0f} |")
