"""echo_gemm_f32 vs cuBLAS (torch, TF32 off) on the fp32 NMT step's GEMM shapes (20 launches captured in a
CUDA graph, CUDA events: no host launch gaps)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1805_08899_b200 import abi
torch.backends.cuda.matmul.allow_tf32 = False
shapes = [(128, 512, 2048, 0, 0, "dh += dA Wh (decoder bwd)"), (128, 2048, 512, 0, 1, "gates += h Wh^T (fwd)"),
          (128, 512, 512, 0, 0, "dctx = dpre Wcc"), (128, 512, 512, 0, 1, "qp = q Wq^T"),
          (2048, 512, 6400, 1, 0, "dWh = dA^T h (wgrad)"), (6400, 2048, 512, 0, 1, "GX = X Wx^T (input proj)"),
          (6400, 512, 2048, 0, 0, "dX = dA Wx"), (6400, 8192, 512, 0, 1, "logits")]
only = sys.argv[1] if len(sys.argv) > 1 else ""
for M, N, K, tA, tB, name in shapes:
    if only and only not in name:
        continue
    A = torch.randn(K, M, device="cuda") if tA else torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda") if tB else torch.randn(K, N, device="cuda")
    C = torch.zeros(M, N, device="cuda")
    opA, opB = (A.t() if tA else A), (B.t() if tB else B)
    lda, ldb = (M if tA else K), (K if tB else N)
    fns = {"cublas": lambda: torch.mm(opA, opB, out=C),
           "echo": lambda: abi.echo_gemm_f32(M, N, K, 1.0, A, lda, tA, B, ldb, tB, 0.0, C, N)}
    res = {}
    for k, f in fns.items():
        for _ in range(3):
            f()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()                       # 20 launches in one graph: no host launch gaps
        with torch.cuda.graph(g):
            for _ in range(20):
                f()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        res[k] = e0.elapsed_time(e1) / 20 * 1e3
    tf = 2 * M * N * K / 1e12
    print(f"{name:28s} M={M:5d} N={N:5d} K={K:5d}  cublas {res['cublas']:8.1f} us ({tf / res['cublas'] * 1e6:5.1f} TF/s)"
          f"  echo {res['echo']:8.1f} us ({tf / res['echo'] * 1e6:5.1f} TF/s)")
