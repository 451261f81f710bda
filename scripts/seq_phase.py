"""Per-phase cycles of the fused LSTM forward (build with ECHO_NVCC_EXTRA=-DECHO_PHASE_TIMING)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_08899_b200 import abi
from paper_1805_08899_b200.lstm import LSTMLayer
B, H, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dt = abi.FP32 if sys.argv[4] == "fp32" else abi.BF16
sd = torch.float32 if dt == abi.FP32 else torch.bfloat16
os.environ["ECHO_LSTM_FUSED"] = "1"
lib = abi.load()
fn = lib.echo_debug_seq_phase
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
X = torch.randn(T, B, H, device="cuda").to(sd)
W = (torch.rand(4 * H, H, device="cuda") * 0.08 - 0.04).to(sd)
b = torch.zeros(4 * H, device="cuda"); h0 = torch.zeros(B, H, device="cuda", dtype=sd); c0 = torch.zeros(B, H, device="cuda")
L = LSTMLayer(T, B, H, dt, abi.RECOMPUTE, "cuda")
L.forward_seq(X, W, W, b, h0, c0); torch.cuda.synchronize()
buf = np.zeros((5, 1024), dtype=np.uint64)
fn(buf.ctypes.data, 1)
L.forward_seq(X, W, W, b, h0, c0); torch.cuda.synchronize()
fn(buf.ctypes.data, 0)
steps = buf[4].max()
n = int((buf[4] > 0).sum())
for i, name in enumerate(["stage h", "gemm", "epilogue", "grid.sync"]):
    v = buf[i, :n].astype(np.float64) / steps
    print(f"{name:10s} mean {v.mean():8.0f} cyc/step  max {v.max():8.0f}")
print("CTAs", n, "steps", steps)
