"""Kernel-time breakdown of one C2 training step (torch.profiler / CUPTI), eager or graph.

    python scripts/profile_step.py [--dtype fp32|bf16] [--mode recompute|stash] [--graph]
Used under ncu as well:  ncu --metrics gpu__time_duration.sum ... python scripts/profile_step.py --ncu
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch

from paper_1805_08899_b200 import abi
from paper_1805_08899_b200.nmt import NMTModel
from synth.configs import C2
from synth.data import nmt_params, nmt_batch

ap = argparse.ArgumentParser()
ap.add_argument("--dtype", default="fp32")
ap.add_argument("--mode", default="recompute")
ap.add_argument("--graph", action="store_true")
ap.add_argument("--ncu", action="store_true", help="no torch profiler; run warm-up then 1 marked step")
ap.add_argument("--batch", type=int, default=128)
args = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = False
dt = abi.FP32 if args.dtype == "fp32" else abi.BF16
md = abi.RECOMPUTE if args.mode == "recompute" else abi.STASH
cfg = C2.with_batch(args.batch)
m = NMTModel(cfg, dt, md)
m.load_params(nmt_params(0, cfg))
m.upload_batch(nmt_batch(1, cfg))
if args.graph:
    m.capture(0.05)
    run = m.replay
else:
    run = lambda: m.step(0.05)
for _ in range(2):
    run()
torch.cuda.synchronize()
if args.ncu:
    torch.cuda.nvtx.range_push("step")
    run()
    torch.cuda.nvtx.range_pop()
    torch.cuda.synchronize()
    sys.exit(0)
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    run()
    torch.cuda.synchronize()
tab = prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=90)
print(tab)
tot = sum(e.device_time_total for e in prof.key_averages())
print("total kernel time (ms):", tot / 1e3)
