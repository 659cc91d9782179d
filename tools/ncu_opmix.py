"""Dynamic SASS opcode mix and stall hot spots of one kernel in an ncu report (source page), here, no GPU.
usage: python tools/ncu_opmix.py report.ncu-rep [per_unit_divisor]"""
import collections
import csv
import io
import subprocess
import sys

path = sys.argv[1]
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter()
stall = collections.Counter()
total = 0
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    n = float(r[ix["Instructions Executed"]] or 0)
    s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    ops[op] += n
    stall[op] += s
    total += n
print(f"total warp instructions {total:.0f} ({total / div:.1f} per unit)")
for op, n in ops.most_common(30):
    print(f"  {op:12s} {n:14.0f} {n / div:10.1f}  {100 * n / total:5.1f}%   stall samples {stall[op]:.0f}")
