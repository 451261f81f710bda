"""Per-step cost of the LSTM recurrence inside a CUDA graph (C2: B = 128, H = 512, bf16): the per-step
path (cuBLAS beta = 1 GEMM + echo_lstm_fwd) vs echo_lstm_fwd_tc (tcgen05 GEMM + fused a1).

    python scripts/lstm_tc_bench.py [--B 128 --H 512 --T 50 --reps 20]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1805_08899_b200 import abi  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--B", type=int, default=128)
ap.add_argument("--H", type=int, default=512)
ap.add_argument("--T", type=int, default=50)
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
B, H, T = a.B, a.H, a.T
bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
gx = (torch.randn(T, B, 4 * H, device="cuda", generator=g) * 0.5).to(bf)
Wh = (torch.randn(4 * H, H, device="cuda", generator=g) / H ** 0.5).to(bf)
bias = torch.randn(4 * H, device="cuda", generator=g) * 0.1
d = abi.LstmDesc(B, H, abi.BF16, abi.RECOMPUTE)


def run(fused):
    gates = gx.clone()
    h = torch.zeros(T + 1, B, H, device="cuda", dtype=bf)
    c = torch.zeros(2, B, H, device="cuda")

    def body():
        for t in range(T):
            if fused:
                abi.echo_lstm_fwd_tc(d, gates[t], h[t], Wh, bias, c[t % 2], gates[t], c[(t + 1) % 2], None, h[t + 1])
            else:
                gates[t].addmm_(h[t], Wh.t())
                abi.echo_lstm_fwd(d, gates[t], None, bias, c[t % 2], gates[t], c[(t + 1) % 2], None, h[t + 1])
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        body()
    torch.cuda.current_stream().wait_stream(s)
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        body()
    for _ in range(3):
        graph.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        graph.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / a.reps / T * 1e3, h[T].float().clone()


us0, h0 = run(False)
us1, h1 = run(True)
print(f"B={B} H={H} T={T}: per-step path {us0:.2f} us/step, tcgen05 fused {us1:.2f} us/step, "
      f"max |h_T diff| {(h0 - h1).abs().max().item():.3e}")
