"""Compact per-kernel table from scripts/profile_step.py --graph output (torch.profiler / CUPTI:
actual in-graph kernel durations, kernels overlapping across streams counted individually).

    python scripts/cupti_summary.py gpurun_out/cupti_c2_fp32_recompute.txt "title" > profiles/x.csv
"""
import re
import sys

src = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else ""
rows = []
unit = {"us": 1.0, "ms": 1e3, "s": 1e6}
for line in open(src):
    parts = re.split(r"\s{2,}", line.strip())
    if len(parts) < 11 or parts[0] in ("Name",) or parts[0].startswith("-"):
        continue
    name, self_cuda, calls = parts[0], parts[6], parts[10]
    m = re.match(r"([\d.]+)(us|ms|s)$", self_cuda)
    if not m:
        continue
    rows.append((name, int(calls), float(m.group(1)) * unit[m.group(2)]))
tot = sum(r[2] for r in rows)
echo = sum(r[2] for r in rows if "echo::" in r[0])
print(f"# {title}")
print("# torch.profiler (CUPTI) kernel activity of one CUDA-graph replay of the step; in-graph durations")
print(f"# total kernel time {tot / 1e3:.3f} ms; libecho (echo::*) share {echo / tot:.4f} (top 30 rows listed)")
print("kernel,calls,total_us,mean_us,share")
for n, c, t in sorted(rows, key=lambda r: -r[2])[:30]:
    n = n.replace(",", ";")[:110]
    print(f"{n},{c},{t:.1f},{t / max(c, 1):.2f},{t / tot:.4f}")
