"""Is initcheck blind to cuBLAS's TMA-store epilogues?  A bf16 GEMM (nvjet, UTMASTG epilogue on
sm_100) writes a fresh buffer; a libecho kernel then reads it.  Under
`compute-sanitizer --tool initcheck` a report here means the GEMM's writes were not tracked."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_1805_08899_b200 import abi  # noqa: E402

for dt, sd in ((abi.BF16, torch.bfloat16), (abi.FP32, torch.float32)):
    a = torch.randn(2, 16, device="cuda").to(sd)
    w = torch.randn(64, 16, device="cuda").to(sd)
    out = torch.empty(2, 64, device="cuda", dtype=sd)
    torch.mm(a, w.t(), out=out)                                  # GEMM writes every element of `out`
    d = abi.LstmDesc(2, 16, dt, abi.RECOMPUTE)
    c0 = torch.zeros(2, 16, device="cuda")
    g = torch.empty_like(out)
    c = torch.empty(2, 16, device="cuda")
    h = torch.empty(2, 16, device="cuda", dtype=sd)
    abi.echo_lstm_fwd(d, out, None, None, c0, g, c, None, h)     # reads `out`
    torch.cuda.synchronize()
    print("dtype", dt, "ok", flush=True)
