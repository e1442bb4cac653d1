"""Summarise an ncu report: key metrics + hottest SASS lines.  Usage: ncu_summary.py REP [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


rows = page("details")
h = rows[0]
want = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy", "Registers Per Thread",
        "Theoretical Occupancy", "Warp Cycles Per Issued Instruction", "Eligible Warps Per Scheduler",
        "Avg. Active Threads Per Warp", "Executed Instructions", "Compute (SM) Throughput", "DRAM Throughput",
        "Grid Size", "Dynamic Shared Memory Per Block"]
for r in rows[1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:40s} {d['Metric Value']:>16s} {d.get('Metric Unit', '')}")
raw = page("raw")
d = dict(zip(raw[0], raw[2] if len(raw) > 2 else raw[1]))
for k in ["sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
          "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
          "dram__bytes_read.sum", "dram__bytes_write.sum"]:
    print(f"{k:70s} {d.get(k, '?')}")
src = page("source", ["--print-source", "sass"])
hh = src[1]
ix = {k: i for i, k in enumerate(hh)}
data = src[2:]
ex = [int(r[ix["Instructions Executed"]] or 0) for r in data]
tot = sum(ex)
print("total warp instructions", tot)
order = sorted(range(len(data)), key=lambda i: -ex[i])[:top]
for i in sorted(order):
    r = data[i]
    print(f"{r[ix['Address']][-5:]} {ex[i] / tot * 100:5.2f}% st={r[ix['Warp Stall Sampling (All Samples)']]:>6} {r[ix['Source']]}")
