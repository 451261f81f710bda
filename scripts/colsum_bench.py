"""echo_colsum timing at the C5 bias-gradient shapes (CUDA events, L2 flushed before each launch):
rows = B*T tokens, cols = 4H (LSTM biases) and V (output bias).

    python scripts/colsum_bench.py [--rows 1228800] [--reps 5] [--only fp32|bf16]
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08899_b200 import abi

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=24576 * 50)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--only", default="")
a = ap.parse_args()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for dt, sd in ((abi.FP32, torch.float32), (abi.BF16, torch.bfloat16)):
    name = "fp32" if dt == abi.FP32 else "bf16"
    if a.only and a.only != name:
        continue
    for cols in (2048, 8192):
        if dt == abi.BF16 and cols == 8192:
            continue                                  # dlogits stay fp32 (the CE feature map)
        x = torch.randn(a.rows, cols, device="cuda").to(sd)
        out = torch.empty(cols, device="cuda")
        ref = x.double().sum(0).float()
        ts = []
        for i in range(a.reps + 2):
            flush.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            abi.echo_colsum(x, out, 0)
            e1.record()
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1))
        ms = statistics.mean(ts)
        nb = x.numel() * x.element_size()
        err = (out - ref).abs().max().item() / ref.abs().max().item()
        print(f"colsum {name} rows={a.rows} cols={cols}: {1e3 * ms:9.1f} us  {nb / 1e9:6.2f} GB  "
              f"{nb / (ms / 1e3) / 1e9:7.1f} GB/s  relerr vs fp64 {err:.2e}", flush=True)
        del x
