"""Per CUDA-source-line totals of an ncu report (cuda,sass view): warp-stall samples and executed
warp instructions, top N lines.

    python scripts/ncu_cuda_lines.py report.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = []
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < 8 or r[0] in ("Line No", "Function Name"):
        continue
    if r[2] != "-":                       # sass rows under a line: skip (the line row carries the totals)
        continue
    try:
        agg.append((int(r[4]), int(r[7] or 0), fname, r[0], r[1].strip()))
    except ValueError:
        continue
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
print(f"stall samples {ts}, warp instructions {ti}")
for s, i, f, ln, src in sorted(agg, reverse=True)[:N]:
    print(f"{100 * s / ts:5.1f}% samp {100 * i / ti:5.1f}% inst  {f}:{ln}  {src[:80]}")
