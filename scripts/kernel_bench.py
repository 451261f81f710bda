"""Per-kernel timing of the hot-path kernels at C2 launch configurations (CUDA events, L2 flushed
before every launch), with algorithmic bytes per launch and achieved GB/s.

    python scripts/kernel_bench.py [--dtype fp32|bf16] [--batch 128] [--only attn_bwd] [--reps 20]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08899_b200 import abi

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--batch", type=int, default=128)
ap.add_argument("--T", type=int, default=50)
ap.add_argument("--H", type=int, default=512)
ap.add_argument("--only", default="")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--noflush", action="store_true")
args = ap.parse_args()
dt = abi.FP32 if args.dtype == "fp32" else abi.BF16
sd = torch.float32 if dt == abi.FP32 else torch.bfloat16
s = 4 if dt == abi.FP32 else 2
B, T, H = args.batch, args.T, args.H
A = Hk = H
Ts = T
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
g = torch.Generator(device="cuda").manual_seed(0)
rn = lambda *sh, sc=1.0: (torch.randn(*sh, device="cuda", generator=g) * sc)


def timeit(fn):
    for _ in range(3):
        fn()
    ts = []
    for _ in range(args.reps):
        if not args.noflush:
            flush.sum()          # read-flush: L2 ends up holding clean lines (no write-back during the timed launch)
        torch.cuda._sleep(200000)  # keep the GPU busy while the host enqueues e0 / launch / e1 (no launch gap timed)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.mean(ts)


res = {}


def report(name, ms, nbytes):
    res[name] = {"us": 1e3 * ms, "bytes": nbytes, "GBps": nbytes / (ms / 1e3) / 1e9}
    print(f"{name:28s} {1e3 * ms:9.2f} us  {nbytes / 1e6:9.2f} MB  {nbytes / (ms / 1e3) / 1e9:8.1f} GB/s", flush=True)


def want(n):
    return not args.only or args.only in n


# ---- LSTM (RECOMPUTE descriptors; STASH for a1/a3 stash variants)
BH = B * H
gates = rn(T, B, 4 * H, sc=0.5).to(sd)
c0 = rn(B, H)
cws = torch.empty(T, B, H, device="cuda")
for md, mname in ((abi.RECOMPUTE, "recompute"), (abi.STASH, "stash")):
    d = abi.LstmDesc(B, H, dt, md)
    gx = rn(B, 4 * H).to(sd)
    gts = torch.empty_like(gx)
    cp = rn(B, H)
    co = torch.empty(B, H, device="cuda")
    tc = torch.empty(B, H, device="cuda", dtype=sd) if md == abi.STASH else None
    h = torch.empty(B, H, device="cuda", dtype=sd)
    if want("lstm_fwd"):
        ms = timeit(lambda: abi.echo_lstm_fwd(d, gx, None, None, cp, gts, co, tc, h))
        nb = BH * (4 * s + 4 + 4 * s + 4 + s + (s if tc is not None else 0))
        report(f"lstm_fwd a1 ({mname})", ms, nb)
    dh = rn(B, H)
    dc = rn(B, H)
    dA = torch.empty_like(gx)
    if want("lstm_bwd"):
        if md == abi.STASH:
            tcs = rn(B, H).to(sd)
            ms = timeit(lambda: abi.echo_lstm_bwd_recompute(d, 1, 0, 0, gts, cp, None, tcs, dh, dc, dA, None, None))
            nb = BH * (4 * s + 4 + s + 4 + 2 * 4 + 4 * s)
        else:
            hr = torch.empty(B, H, device="cuda", dtype=sd)
            ms = timeit(lambda: abi.echo_lstm_bwd_recompute(d, 1, 0, 0, gts, cp, None, None, dh, dc, dA, hr, co))
            nb = BH * (4 * s + 4 + 4 + 4 + 2 * 4 + 4 * s + s)
        report(f"lstm_bwd a3 ({mname})", ms, nb)
if want("cscan"):
    d = abi.LstmDesc(B, H, dt, abi.RECOMPUTE)
    ms = timeit(lambda: abi.echo_lstm_cscan(d, T, gates, c0, cws, None))
    report("lstm_cscan a2", ms, T * BH * (3 * s + 4) + BH * 4)

# ---- attention (s-major layout as in the NMT step)
qp = rn(B, A, sc=0.5).to(sd)
Kp = rn(Ts, B, A, sc=0.5).to(sd)
Hs = rn(Ts, B, Hk).to(sd)
v = rn(A, sc=0.1).to(sd)
sl = torch.full((B,), Ts, dtype=torch.int32, device="cuda")
dctx = rn(B, Hk)
ctx = torch.empty(B, Hk, device="cuda", dtype=sd)
rows = B * Ts
for md, mname in ((abi.RECOMPUTE, "recompute"), (abi.STASH, "stash")):
    d = abi.AttnDesc(B, Ts, A, Hk, dt, md, A, B * A, Hk, B * Hk)
    Z = torch.empty(B, Ts, A, device="cuda", dtype=sd) if md == abi.STASH else None
    al = torch.empty(B, Ts, device="cuda") if md == abi.STASH else None
    if want("attn_fwd"):
        ms = timeit(lambda: abi.echo_attn_fwd(d, qp, Kp, v, Hs, sl, ctx, Z, al))
        nb = rows * (A * s + Hk * s) + (rows * (A * s + 4) if md == abi.STASH else 0) + B * (A + Hk) * s
        report(f"attn_fwd a5 ({mname})", ms, nb)
    abi.echo_attn_fwd(d, qp, Kp, v, Hs, sl, ctx, Z, al)
    dqp = torch.empty(B, A, device="cuda")
    dKp = torch.zeros(Ts, B, A, device="cuda")
    dHs = torch.zeros(Ts, B, Hk, device="cuda")
    dvp = torch.zeros(B, A, device="cuda")
    creg = torch.empty(B, Hk, device="cuda", dtype=sd) if md == abi.RECOMPUTE else None
    if want("attn_bwd"):
        if md == abi.RECOMPUTE:
            ms = timeit(lambda: abi.echo_attn_bwd_recompute(d, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, None, creg, dvp))
            nb = rows * (A * s + Hk * s + 2 * A * 4 + 2 * Hk * 4)
        else:
            ms = timeit(lambda: abi.echo_attn_bwd_recompute(d, None, None, v, Hs, sl, Z, al, dctx, dqp, dKp, dHs, None, None, dvp))
            nb = rows * (A * s + 4 + Hk * s + 2 * A * 4 + 2 * Hk * 4)
        nb += B * A * s + B * Hk * 4 + B * A * 4 + 2 * B * A * 4 + B * Hk * s
        report(f"attn_bwd a6 ({mname})", ms, nb)
print(json.dumps(res))
