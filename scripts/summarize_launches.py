"""Summarise an ncu launch list (gpu__time_duration.sum, --csv) into per-kernel totals and shares.

    python scripts/summarize_launches.py gpurun_out/launches_fp32.csv profiles/r01_launches.csv "title"
"""
import collections
import csv
import re
import sys

src, dst = sys.argv[1], sys.argv[2]
title = sys.argv[3] if len(sys.argv) > 3 else ""
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hi]
ki, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    try:
        us = float(r[vi].replace(",", "")) * scale[r[ui]]
    except (ValueError, KeyError):
        continue
    name = re.sub(r"\(.*", "", r[ki]).replace("void ", "")[:100]
    agg[name][0] += 1
    agg[name][1] += us
tot = sum(v[1] for v in agg.values())
n = sum(v[0] for v in agg.values())
echo = sum(v[1] for k, v in agg.items() if k.startswith("echo::"))
out = [f"# {title}",
       "# ncu --metrics gpu__time_duration.sum --clock-control none (serialised, cold cache per launch:",
       "# compare SHARES, not absolutes)",
       f"# total kernel time {tot / 1e3:.3f} ms over {n} launches; libecho (echo::*) share {echo / tot:.4f}",
       "kernel,launches,total_us,mean_us,share"]
for k, (c, us) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.append(f"{k.replace(',', ';')},{c},{us:.1f},{us / c:.2f},{us / tot:.4f}")
open(dst, "w").write("\n".join(out) + "\n")
print("\n".join(out[:30]))
