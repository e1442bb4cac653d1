"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into a markdown table.

usage: python tools/launch_list.py LAUNCHES.csv "COMMAND" > profiles/<name>.md
"""
import csv
import sys
from collections import defaultdict

path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
rows = []
with open(path) as fh:
    lines = [ln for ln in fh if ln.startswith('"')]
for r in csv.DictReader(lines):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        rows.append((r["Kernel Name"], float(r["Metric Value"].replace(",", "")), r["Metric Unit"]))
units = sorted({u for _, _, u in rows})
scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0, "nsecond": 1e-6}
agg = defaultdict(lambda: [0, 0.0])
for name, v, u in rows:
    agg[name][0] += 1
    agg[name][1] += v * scale.get(u, 1e-6)
total = sum(t for _, t in agg.values()) or 1.0
print(f"# ncu launch list: `{cmd}`\n")
print("`ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised per launch: "
      f"compare SHARES). Raw units reported by ncu: {units}.\n")
print("| kernel | launches | total | avg per launch | share |")
print("|---|---|---|---|---|")
for name, (cnt, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    short = name.split("(")[0][:70]
    print(f"| `{short}` | {cnt} | {t:.2f} ms | {t / cnt * 1e3:.1f} us | {t / total * 100:.1f}% |")
