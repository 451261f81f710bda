"""Hot SASS instructions of an ncu report (source page, SASS view): top-N by warp-stall samples, and
a coarse breakdown of samples / executed instructions by mnemonic class.

    python scripts/ncu_sass_hot.py report.ncu-rep [N]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ix = {n: i for i, n in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        data.append((int(r[ix["Warp Stall Sampling (All Samples)"]]), int(r[ix["Instructions Executed"]] or 0),
                     r[ix["Address"]][-5:], r[ix["Source"]].strip()))
    except ValueError:
        continue
tot = sum(d[0] for d in data)
ins = sum(d[1] for d in data)
print(f"total stall samples {tot}, warp instructions executed {ins}")
cls = collections.Counter()
cli = collections.Counter()
for s, n, a, src in data:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    cls[op] += s
    cli[op] += n
print("by mnemonic (samples %, instr %):")
for op, s in cls.most_common(25):
    print(f"  {op:10s} {100 * s / tot:5.1f}%  {100 * cli[op] / max(ins, 1):5.1f}%")
print(f"top {N} instructions:")
for s, n, a, src in sorted(data, reverse=True)[:N]:
    print(f"  {100 * s / tot:5.1f}%  {n:>10d}  {a}  {src[:90]}")
