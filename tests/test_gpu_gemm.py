"""libecho's IEEE-fp32 split-K GEMM (echo_gemm_f32, row a0) vs an fp64 reference of the same op;
deterministic (bitwise run-to-run) and fp32-accurate (no TF32)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 512, 2048), (128, 2048, 512), (128, 512, 512), (6400, 512, 2048),
                                   (2048, 512, 6400), (5, 52, 20), (1, 4, 4), (300, 1000, 772)])
@pytest.mark.parametrize("tA,tB", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("beta", [0.0, 1.0])
def test_gemm_f32(M, N, K, tA, tB, beta, cuda_dev):
    from paper_1805_08899_b200 import abi
    lda = M if tA else K
    ldb = K if tB else N
    if not abi.echo_gemm_f32_supported(M, N, K, tA, tB, lda, ldb, N):
        pytest.skip("shape outside the fast path (caller falls back to cuBLAS)")
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N + K)
    A = torch.randn(K, M, device="cuda", generator=g) if tA else torch.randn(M, K, device="cuda", generator=g)
    B = torch.randn(N, K, device="cuda", generator=g) if tB else torch.randn(K, N, device="cuda", generator=g)
    C0 = torch.randn(M, N, device="cuda", generator=g)
    C = C0.clone()
    abi.echo_gemm_f32(M, N, K, 1.0, A, lda, tA, B, ldb, tB, beta, C, N)
    Ad = (A.t() if tA else A).double()
    Bd = (B.t() if tB else B).double()
    ref = Ad @ Bd + beta * C0.double()
    err = (C.double() - ref).abs().max().item()
    scale = (Ad.abs() @ Bd.abs()).max().item() + beta * C0.abs().max().item()
    assert err <= 4 * K * 2 ** -24 * scale, (err, scale)            # fp32 FMA-chain bound (no TF32)
    C2 = C0.clone()
    abi.echo_gemm_f32(M, N, K, 1.0, A, lda, tA, B, ldb, tB, beta, C2, N)
    assert torch.equal(C, C2)


def test_gemm_wrapper_routes_views(cuda_dev):
    """gemm.mm / addmm_ on transposed views (W.t()) go through echo_gemm_f32 and match torch."""
    from paper_1805_08899_b200 import gemm
    torch.backends.cuda.matmul.allow_tf32 = False
    saved = gemm._MODE
    gemm._MODE = "echo"
    x = torch.randn(128, 512, device="cuda")
    W = torch.randn(2048, 512, device="cuda")
    c = torch.randn(128, 2048, device="cuda")
    r = torch.addmm(c, x, W.t())
    gemm.addmm_(c, x, W.t())
    assert (c - r).abs().max().item() <= 1e-3
    y = gemm.mm(x.t().contiguous().t(), W.t())
    assert (y - x @ W.t()).abs().max().item() <= 1e-3
    gemm._MODE = saved
