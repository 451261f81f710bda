"""Fused persistent LSTM forward (echo_lstm_seq_fwd) vs the per-step path (cuBLAS GEMM + a1):
per-step time of one layer, CUDA events, warm.

    python scripts/seq_bench.py [--B 128 --H 512 --T 50 --dtype fp32]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1805_08899_b200 import abi
from paper_1805_08899_b200.lstm import LSTMLayer

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--H", type=int, default=512)
ap.add_argument("--T", type=int, default=50)
ap.add_argument("--dtype", default="fp32")
args = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = False
dt = abi.FP32 if args.dtype == "fp32" else abi.BF16
sd = torch.float32 if dt == abi.FP32 else torch.bfloat16
T, B, H = args.T, args.B, args.H
g = torch.Generator(device="cuda").manual_seed(0)
X = torch.randn(T, B, H, device="cuda", generator=g).to(sd)
Wx = (torch.rand(4 * H, H, device="cuda", generator=g) * 0.08 - 0.04).to(sd)
Wh = (torch.rand(4 * H, H, device="cuda", generator=g) * 0.08 - 0.04).to(sd)
b = torch.zeros(4 * H, device="cuda")
h0 = torch.zeros(B, H, device="cuda", dtype=sd)
c0 = torch.zeros(B, H, device="cuda")
for flag in ("0", "1"):
    os.environ["ECHO_LSTM_FUSED"] = flag
    L = LSTMLayer(T, B, H, dt, abi.RECOMPUTE, "cuda")
    for _ in range(3):
        L.forward_seq(X, Wx, Wh, b, h0, c0)
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        L.forward_seq(X, Wx, Wh, b, h0, c0)
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"{args.dtype} B={B} H={H} T={T} fused={flag}: layer {ms * 1e3:.1f} us = {ms * 1e3 / T:.2f} us/step "
          f"(incl. the input-projection GEMM)")
