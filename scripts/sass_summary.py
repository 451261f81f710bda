"""Static SASS summary of libecho kernels (no GPU): registers / stack / shared from cuobjdump's resource
usage, and counts of the instructions that prove the design (TMA loads UTMALDG / UBLKCP, mbarrier
SYNCS, tcgen05 UTC*MMA / LDTM, packed fp32 FFMA2 / FMUL2 / FADD2, bf16x2 HADD2 / HFMA2, MUFU,
global / shared vector accesses).

    python scripts/sass_summary.py [regex] > profiles/r02_sass_summary.txt
"""
import collections
import re
import subprocess
import sys

LIB = "paper_1805_08899_b200/libecho.so"
CUOBJDUMP = "/usr/local/cuda/bin/cuobjdump"
pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else r"attn_fwd_rows|attn_fwd_tma|attn_bwd_tma|lstm_cscan|lstm_fwd_tc")
KEYS = ["UTMALDG", "UTMAPF", "UBLKCP", "SYNCS", "UTCHMMA", "UTCBAR", "LDTM", "FFMA2", "FMUL2", "FADD2", "HADD2",
        "HFMA2", "MUFU", "LDG.E.128", "STG.E.128", "LDS.128", "LDS.64", "SHFL", "BAR.SYNC", "NANOSLEEP", "BPT.TRAP"]

res = subprocess.run([CUOBJDUMP, "--dump-resource-usage", LIB], capture_output=True, text=True).stdout
usage = {}
fn = None
for line in res.splitlines():
    m = re.search(r"Function (\S+):", line)
    if m:
        fn = m.group(1)
    m = re.search(r"REG:(\d+) STACK:(\d+) SHARED:(\d+) LOCAL:(\d+)", line)
    if m and fn:
        usage[fn] = tuple(int(x) for x in m.groups())
sass = subprocess.run([CUOBJDUMP, "-sass", LIB], capture_output=True, text=True).stdout
counts, cur = {}, None
for line in sass.splitlines():
    m = re.match(r"\s+Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", line)
    if cur and m:
        op = m.group(1)
        counts[cur]["total"] += 1
        for k in KEYS:
            if op.startswith(k):
                counts[cur][k] += 1
print("# static SASS summary of libecho.so (sm_100a): resource usage and key instruction counts per kernel")
print("# (HFMA2 counts include the compiler's HFMA2.MMA register-move idiom; SYNCS = mbarrier init / arrive / try-wait)")
print("# kernel | REG STACK SHARED(static) LOCAL | SASS instructions | " + " ".join(KEYS))
for k in sorted(counts):
    dm = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    if not pat.search(dm):
        continue
    u = usage.get(k, (0, 0, 0, 0))
    c = counts[k]
    print(f"{dm[:110]} | {u[0]} {u[1]} {u[2]} {u[3]} | {c['total']} | " + " ".join(f"{x}={c[x]}" for x in KEYS if c[x]))
