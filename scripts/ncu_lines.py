"""Per-source-line warp-stall samples and executed warp instructions from an ncu report
(`--import-source on`, compiled with -lineinfo).

    python scripts/ncu_lines.py gpurun_out/x.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_i = hdr.index("Instructions Executed")
lines = []
for r in rows:
    if r and r[0].isdigit():
        try:
            lines.append((int(r[i_s]), int(r[i_i]), int(r[0]), r[1].strip()))
        except ValueError:
            pass
tot_s = sum(x[0] for x in lines) or 1
tot_i = sum(x[1] for x in lines) or 1
print(f"# {rep.split('/')[-1]}: {tot_s} stall samples, {tot_i} warp instructions executed")
print(f"{'samples%':>8} {'inst%':>6}  line  source")
for s, i, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{100 * s / tot_s:8.1f} {100 * i / tot_i:6.1f}  {ln:4d}  {src[:90]}")
