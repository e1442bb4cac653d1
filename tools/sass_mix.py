"""Instruction mix from an exported ncu SASS source page (tools/ncu_export.sh): executed warp
instructions per opcode, and per competitor-timestep when ct is given.
usage: python tools/sass_mix.py REPORT.source.csv.gz [ct] [top]"""
import collections
import csv
import gzip
import io
import sys

path = sys.argv[1]
ct = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
with gzip.open(path, "rt") as fh:
    rows = list(csv.reader(io.StringIO(fh.read())))
hdr_i = next(i for i, r in enumerate(rows) if "Source" in r and "Instructions Executed" in r)
h = rows[hdr_i]
ix = {k: i for i, k in enumerate(h)}
mix = collections.Counter()
tot = 0
for r in rows[hdr_i + 1:]:
    if len(r) < len(h):
        continue
    try:
        ex = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    src = r[ix["Source"]].strip()
    if src.startswith("@"):
        src = src.split(None, 1)[1] if " " in src else src
    op = src.split()[0] if src else "?"
    mix[op] += ex
    tot += ex
print(f"total warp instructions {tot:.4g}" + (f"  per ct {tot / ct:.3f}" if ct else ""))
for op, v in mix.most_common(top):
    print(f"{op:28s} {v / tot * 100:6.2f}%" + (f"  {v / ct:.4f}/ct" if ct else ""))
