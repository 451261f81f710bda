"""One small NMT / attention workload for compute-sanitizer (memcheck, racecheck, synccheck, initcheck):
the full training step (encoder wavefront on two streams, a5/a6 TMA + DSMEM kernels, LSTM a1/a2/a3,
fused CE, colsum) in both modes, eagerly and as a CUDA-graph replay, plus a standalone attention
call at the C2 row shape.

    compute-sanitizer --tool racecheck --error-exitcode 9 python scripts/sanitize_step.py --cfg c1
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1805_08899_b200 import abi  # noqa: E402
from paper_1805_08899_b200.nmt import NMTModel  # noqa: E402
from synth.configs import C1, SMALL_NMT  # noqa: E402
from synth.data import nmt_params, nmt_batch  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", default="c1", choices=["c1", "small"])
ap.add_argument("--dtype", default="fp32", choices=["fp32", "bf16"])
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = False
cfg = C1 if a.cfg == "c1" else SMALL_NMT
dt = abi.FP32 if a.dtype == "fp32" else abi.BF16
P, B = nmt_params(1, cfg, a.dtype), nmt_batch(2, cfg, lengths="random")
for mode in (abi.STASH, abi.RECOMPUTE):
    m = NMTModel(cfg, dt, mode)
    m.load_params(P)
    m.upload_batch(B)
    m.step(0.0)                                               # eager
    if not a.no_graph:
        m.capture(0.0, warmup=1)                              # + CUDA-graph replay
        m.replay()
    torch.cuda.synchronize()
    print(f"mode {mode}: loss {float(m.loss):.6f}", flush=True)
# one attention forward / backward at a C2-like row (Ts = 50, A = Hk = 512: 4-CTA clusters)
Bq, Ts, A = 3, 50, 512
sd = torch.float32 if dt == abi.FP32 else torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
Kp = torch.randn(Ts, Bq, A, device="cuda", generator=g).to(sd)
Hs = torch.randn(Ts, Bq, A, device="cuda", generator=g).to(sd)
qp = torch.randn(Bq, A, device="cuda", generator=g).to(sd)
v = torch.randn(A, device="cuda", generator=g).to(sd)
sl = torch.tensor([50, 17, 1], dtype=torch.int32, device="cuda")
d = abi.AttnDesc(Bq, Ts, A, A, dt, abi.RECOMPUTE, A, Bq * A, A, Bq * A)
ctx = torch.empty(Bq, A, device="cuda", dtype=sd)
abi.echo_attn_fwd(d, qp, Kp, v, Hs, sl, ctx, None, None)
dctx = torch.randn(Bq, A, device="cuda", generator=g)
dqp = torch.empty(Bq, A, device="cuda")
dKp = torch.zeros(Ts, Bq, A, device="cuda")
dHs = torch.zeros(Ts, Bq, A, device="cuda")
ws = torch.zeros(Bq, A, device="cuda")
dv = torch.empty(A, device="cuda")
creg = torch.empty_like(ctx)
abi.echo_attn_bwd_recompute(d, qp, Kp, v, Hs, sl, None, None, dctx, dqp, dKp, dHs, dv, creg, ws)
torch.cuda.synchronize()
assert torch.equal(creg.view(torch.uint8), ctx.view(torch.uint8))
print("attention ok", flush=True)
