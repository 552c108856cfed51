"""Summarise an ncu report (``--set full``) or a launch-list CSV into a
markdown table for profiles/.

    python tools/ncu_summary.py gpurun_out/r1_full.ncu-rep > profiles/r1_ncu_full.md
    python tools/ncu_summary.py --launches gpurun_out/launches_r1.csv > profiles/r1_launches.md
"""

from __future__ import annotations

import argparse
import collections
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", "DRAM rd"),
    ("dram__bytes_write.sum", "DRAM wr"),
    ("lts__t_sector_hit_rate.pct", "L2 hit %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM %"),
    ("sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed", "tensor %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
]
STALLS = ["long_scoreboard", "barrier", "short_scoreboard", "wait", "mio_throttle", "lg_throttle",
          "math_pipe_throttle", "selected", "not_selected", "dispatch_stall", "branch_resolving"]


def _short(name: str) -> str:
    return name.split("(")[0].split("::")[-1]


def _num(v: str) -> float:
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return float("nan")


def full(path: str) -> str:
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(head)}
    for n, i in list(col.items()):  # section-prefixed copies ("TPC.TriageCompute.<metric>")
        col.setdefault(n.split(".", 2)[-1] if n.count(".") >= 3 and not n[0].islower() else n, i)
    out = [f"# ncu --set full summary of `{path.split('/')[-1]}`", "",
           "One launch per kernel, cold-cache and serialised under the profiler (absolute times are",
           "not bench numbers; the share of the step and the limiters are what this is for).", ""]
    names = [m for m, _ in METRICS if m in col]
    out.append("| kernel | " + " | ".join(dict(METRICS)[m] + (f" ({units[col[m]]})" if units[col[m]] else "")
                                          for m in names) + " | DRAM GB/s |")
    out.append("|---" * (len(names) + 2) + "|")
    for r in data:
        gbs = ((_num(r[col["dram__bytes_read.sum"]]) + _num(r[col["dram__bytes_write.sum"]]))
               / _num(r[col["gpu__time_duration.sum"]]) * 1e3)  # Gbyte / ms
        out.append(f"| {_short(r[col['Kernel Name']])} | " + " | ".join(r[col[m]] for m in names)
                   + f" | {gbs:.0f} |")
    out += ["", "Warp stall samples (smsp__pcsamp_warps_issue_stalled_*), % of the kernel's samples:", ""]
    scols = {s: col.get("smsp__pcsamp_warps_issue_stalled_" + s) for s in STALLS}
    out.append("| kernel | " + " | ".join(STALLS) + " |")
    out.append("|---" * (len(STALLS) + 1) + "|")
    for r in data:
        vals = {s: _num(r[c]) if c is not None else 0.0 for s, c in scols.items()}
        tot = sum(v for v in vals.values() if v == v) or 1.0
        out.append(f"| {_short(r[col['Kernel Name']])} | " +
                   " | ".join(f"{100 * vals[s] / tot:.0f}" for s in STALLS) + " |")
    return "\n".join(out) + "\n"


def launches(path: str) -> str:
    text = open(path).read()
    start = text.find('"ID"')  # skip the ==PROF== preamble
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    agg = collections.OrderedDict()
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = _short(r["Kernel Name"])
        v = _num(r["Metric Value"])
        unit = r.get("Metric Unit", "")
        ms = v / 1e6 if unit == "ns" else v / 1e3 if unit in ("us", "usecond") else v
        n, t = agg.get(k, (0, 0.0))
        agg[k] = (n + 1, t + ms)
    total = sum(t for _, t in agg.values()) or 1.0
    out = [f"# ncu launch list `{path.split('/')[-1]}` (gpu__time_duration.sum, --clock-control none)", "",
           "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| {k} | {n} | {t:.3f} | {100 * t / total:.1f}% |")
    out.append(f"| **all** | {sum(n for n, _ in agg.values())} | {total:.3f} | 100% |")
    return "\n".join(out) + "\n"


def main(argv=None) -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("path")
    ap.add_argument("--launches", action="store_true")
    a = ap.parse_args(argv)
    sys.stdout.write(launches(a.path) if a.launches else full(a.path))


if __name__ == "__main__":
    main()
