"""In-step hot-path kernel times (probe.py: timing events inside the step's CUDA graph) for a
workload and mode: per kernel launches/step, mean us, total ms/step and share of the step.

    python scripts/step_kernels.py [--cfg C2|C3|C4] [--dtype fp32|bf16] [--steps 5] [--json out]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08899_b200 import abi
from synth import configs as K
from synth import data as D

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="C2")
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--steps", type=int, default=5)
ap.add_argument("--json", default="")
args = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = False
dt = abi.FP32 if args.dtype == "fp32" else abi.BF16
if args.cfg == "C2":
    from paper_1805_08899_b200.nmt import NMTModel as M
    cfg = K.C2
    params, batch = D.nmt_params(0, cfg, args.dtype), D.nmt_batch(1, cfg)
elif args.cfg == "C3":
    from paper_1805_08899_b200.ds2 import DS2Model as M
    cfg = K.C3
    params, batch = D.ds2_params(0, cfg, args.dtype), D.ds2_batch(1, cfg, args.dtype)
else:
    from paper_1805_08899_b200.transformer import TXModel as M
    cfg = K.C4
    params, batch = D.tx_params(0, cfg, args.dtype), D.tx_batch(1, cfg, args.dtype)
res = {"cfg": args.cfg, "dtype": args.dtype}
for mode, name in ((abi.STASH, "stash"), (abi.RECOMPUTE, "recompute")):
    m = M(cfg, dt, mode)
    m.load_params(params)
    m.upload_batch(batch)
    m.capture(0.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        m.replay()
    e0.record()
    for _ in range(args.steps):
        m.replay()
    e1.record()
    torch.cuda.synchronize()
    plain = e0.elapsed_time(e1) / args.steps
    m.capture(0.0, with_probe=True)
    per, tot = {}, 0.0
    for _ in range(args.steps):
        e0.record()
        m.replay()
        e1.record()
        for k, v in m.kernel_times().items():
            per.setdefault(k, []).extend(v)
        tot += e0.elapsed_time(e1)
    probed = tot / args.steps
    rows = {}
    for k, v in sorted(per.items()):
        n = len(v) // args.steps
        rows[k] = {"launches": n, "mean_us": 1e3 * statistics.mean(v), "ms_per_step": sum(v) / args.steps}
    hot = sum(r["ms_per_step"] for r in rows.values())
    res[name] = {"step_ms": plain, "probed_step_ms": probed, "kernels": rows, "hot_ms": hot, "hot_share": hot / probed}
    print(f"== {args.cfg} {args.dtype} {name}: step {plain:.3f} ms (probed {probed:.3f}); hot-path kernels "
          f"{hot:.3f} ms = {100 * hot / probed:.1f}%")
    for k, r in rows.items():
        print(f"   {k:12s} {r['launches']:5d} x {r['mean_us']:8.2f} us = {r['ms_per_step']:7.3f} ms")
    del m
    torch.cuda.empty_cache()
if args.json:
    json.dump(res, open(args.json, "w"), indent=1)
