"""Markdown table of single-launch ncu captures (tools/ncu_tail.sh):
duration, grid, cluster, DRAM bytes, top stall reasons.
    python tools/ncu_tail_table.py gpurun_out/tailB_*.ncu-rep"""
import csv
import io
import subprocess
import sys

print("| kernel | grid | cluster | duration µs | DRAM MB | warps active % | issue % | tensor pipe % | top stalls |")
print("|---|---|---|---|---|---|---|---|---|")
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        continue
    h, units = rows[0], dict(zip(rows[0], rows[1]))
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    for r in rows[2:]:
        d = dict(zip(h, r))
        st = {k: float(v.replace(",", "")) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued") and v}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda x: -x[1])[:3]
        stalls = ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.0f}%" for k, v in top)
        def num(k):
            v = d.get(k)
            if v is None:   # some metrics carry a section prefix in the raw page
                v = next((x for h_, x in d.items() if h_.endswith("." + k)), "")
            try:
                return float(v.replace(",", ""))
            except ValueError:
                return float("nan")
        name = d["Kernel Name"].split("(")[0].replace("<unnamed>::", "").replace("void ", "")
        mb = sum(num(k) * scale.get(units.get(k, "Mbyte"), 1.0) for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"))
        print(f"| {name} | {d.get('launch__grid_size')} | {d.get('launch__cluster_dim_x', '') or '-'} | "
              f"{num('gpu__time_duration.sum') * {'ns': 1e-3, 'us': 1.0, 'ms': 1e3, 'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3}.get(units.get('gpu__time_duration.sum'), 1.0):.1f} | {mb:.1f} | "
              f"{num('sm__warps_active.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{num('smsp__issue_active.avg.pct_of_peak_sustained_active'):.0f} | "
              f"{num('sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed'):.0f} | {stalls} |")
