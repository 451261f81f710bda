"""Text summary of an `ncu --set full` report: launch config, duration, DRAM traffic, throughput,
occupancy, top stall reasons and the top stalled SASS lines.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [algorithmic_bytes] > profiles/x.txt
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
alg = float(sys.argv[2]) if len(sys.argv) > 2 else None


def page(p, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", p, "--csv", *extra], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("raw")
hdr, vals = raw[0], raw[2] if len(raw) > 2 else raw[1]
d = dict(zip(hdr, vals))
keys = ["Kernel Name", "launch__grid_size", "launch__block_size", "launch__cluster_dim_x", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum"]
units = raw[1] if len(raw) > 2 else [""] * len(hdr)
u = dict(zip(hdr, units))
print(f"# ncu --set full summary of {rep.split('/')[-1]}")
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k]} {u.get(k, '')}")


def num(k):
    try:
        return float(d[k].replace(",", ""))
    except (KeyError, ValueError):
        return None


def to_bytes(k):
    v = num(k)
    if v is None:
        return None
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)


rd, wr = to_bytes("dram__bytes_read.sum"), to_bytes("dram__bytes_write.sum")
if rd is not None and wr is not None:
    print(f"{'traffic = dram read + write (bytes)':70s} {rd + wr:.0f}")
    if alg:
        print(f"{'algorithmic bytes per launch':70s} {alg:.0f}   traffic/algorithmic = {(rd + wr) / alg:.3f}")
stalls = sorted(((k, num(k)) for k in d if k.startswith("smsp__average_warps_issue_stalled") and k.endswith("per_issue_active.ratio")),
                key=lambda x: -(x[1] or 0))
print("# top warp stall reasons (warps per issued instruction)")
for k, v in stalls[:8]:
    print(f"  {k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):30s} {v}")
src = page("source", ("--print-source", "sass"))
if len(src) > 2:
    h = src[1]
    if "Warp Stall Sampling (All Samples)" in h:
        i_s = h.index("Warp Stall Sampling (All Samples)")
        rows = src[2:]
        tot = sum(float(r[i_s] or 0) for r in rows) or 1.0
        print(f"# top stalled SASS instructions ({tot:.0f} samples)")
        for r in sorted(rows, key=lambda r: -float(r[i_s] or 0))[:15]:
            print(f"  {float(r[i_s]) / tot * 100:5.1f}%  {r[1][:100]}")
