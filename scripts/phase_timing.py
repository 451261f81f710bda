"""Per-phase cycle breakdown of attn_bwd_tma (needs a build with ECHO_NVCC_EXTRA=-DECHO_PHASE_TIMING)."""
import ctypes, sys, os, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1805_08899_b200 import abi
B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
Ts, A, H = 50, 512, 512
lib = abi.load()
fn = lib.echo_debug_phase_times
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
g = torch.Generator(device="cuda").manual_seed(0)
rn = lambda *s, sc=1.0: torch.randn(*s, device="cuda", generator=g) * sc
qp, Kp, Hs, v = rn(B, A, sc=.5), rn(Ts, B, A, sc=.5), rn(Ts, B, H), rn(A, sc=.1)
sl = torch.full((B,), Ts, dtype=torch.int32, device="cuda")
dctx = rn(B, H); dqp = torch.empty(B, A, device="cuda"); dKp = torch.zeros(Ts, B, A, device="cuda")
dHs = torch.zeros(Ts, B, H, device="cuda"); dvp = torch.zeros(B, A, device="cuda"); creg = torch.empty(B, H, device="cuda")
d = abi.AttnDesc(B, Ts, A, H, abi.FP32, abi.RECOMPUTE, A, B * A, H, B * H)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for _ in range(3):
    abi.echo_attn_bwd_recompute(d, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, None, creg, dvp)
flush.sum(); torch.cuda._sleep(200000)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); abi.echo_attn_bwd_recompute(d, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, None, creg, dvp); e1.record(); e1.synchronize()
print("kernel ms", e0.elapsed_time(e1))
buf = np.zeros((16, 8192), dtype=np.uint64)
fn(buf.ctypes.data, 16 * 8192)
ncta = B * 4
t = buf[:, :ncta].astype(np.int64)
names = ["start->issued", "issued->tma_done", "tma_done->phase1_end", "phase1->clsync", "clsync->gathered",
         "gathered->softmax", "softmax->ctx", "ctx->phase4_end", "phase4->reduced", "reduced->cluster_wait"]
for k in range(10):
    dd = t[k + 1] - t[k]
    print(f"{names[k]:24s} mean {dd.mean():8.0f} cyc  p50 {np.median(dd):8.0f}  max {dd.max():8.0f}")
print("start->barriers_init    mean", (t[11]-t[0]).mean(), " start->all_issued mean", (t[12]-t[0]).mean())
tot = t[10] - t[0]
print("CTA lifetime cycles mean", tot.mean(), "max", tot.max())
gt = buf[15, :ncta].astype(np.int64); gt -= gt.min()
print("CTA start spread (ns): p50", np.median(gt), "max", gt.max())
ge = buf[14, :ncta].astype(np.int64) - buf[15, :ncta].astype(np.int64).min()
print("globaltimer: first start -> last end (ns)", ge.max(), " per-CTA lifetime ns p50",
      np.median(buf[14, :ncta].astype(np.int64) - buf[15, :ncta].astype(np.int64)))
