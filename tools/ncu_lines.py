"""Per-CUDA-source-line instruction counts from an ncu report (needs -lineinfo + --import-source on).
usage: python tools/ncu_lines.py REPORT [topN]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = {}
cur_file = None
cur_line = None
hdr = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = {k: i for i, k in enumerate(r)}
        continue
    if not hdr or len(r) < 8:
        continue
    if r[0]:
        cur_line = (cur_file, int(r[0]), r[1][:90])
        continue
    try:
        e = int(r[7] or 0)
    except ValueError:
        continue
    agg[cur_line] = agg.get(cur_line, 0) + e
tot = sum(agg.values()) or 1
for (f, ln, src), e in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    print(f"{e / tot * 100:5.1f}%  {f}:{ln:<4d} {src}")
