"""Fused output-layer softmax cross-entropy (echo_xent_fwd_bwd) vs a plain fp64 reference of the
same op (reading R10: mean CE; dLoss/dlogits = (softmax - onehot) / N)."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(x, b, y):
    z = x + (b if b is not None else 0.0)
    m = z.max(axis=1, keepdims=True)
    lse = m[:, 0] + np.log(np.exp(z - m).sum(axis=1))
    rows = lse - z[np.arange(len(y)), y]
    p = np.exp(z - lse[:, None])
    p[np.arange(len(y)), y] -= 1.0
    return rows, p / len(y)


@pytest.mark.parametrize("N,V,bias,copy", [(64, 8192, True, True), (37, 29, True, False), (5, 1000, False, True),
                                           (3000, 128, True, True), (1, 4, False, False)])
def test_xent_matches_reference(N, V, bias, copy, cuda_dev):
    from paper_1805_08899_b200 import abi
    rng = np.random.default_rng(N * 7 + V)
    x = (rng.standard_normal((N, V)) * 3).astype(np.float32)
    b = rng.standard_normal(V).astype(np.float32) if bias else None
    y = rng.integers(0, V, N)
    rows_ref, d_ref = _ref(x.astype(np.float64), None if b is None else b.astype(np.float64), y)
    lg = torch.from_numpy(x).cuda()
    bb = torch.from_numpy(b).cuda() if bias else None
    yy = torch.from_numpy(y).cuda()
    rl = torch.empty(N, device="cuda")
    cp = torch.empty(N, V, dtype=torch.bfloat16, device="cuda") if copy else None
    abi.echo_xent_fwd_bwd(N, V, lg, bb, yy, rl, cp)
    torch.cuda.synchronize()
    rows, d = rl.cpu().numpy(), lg.cpu().numpy()
    assert np.max(np.abs(rows - rows_ref)) <= 1e-4 * np.max(np.abs(rows_ref))
    assert np.max(np.abs(d - d_ref)) <= 1e-4 * np.max(np.abs(d_ref))
    assert np.allclose(d.sum(axis=1), 0.0, atol=1e-6)               # softmax - onehot sums to 0
    if copy:
        assert torch.equal(cp, torch.from_numpy(d).cuda().to(torch.bfloat16))
    # deterministic: a second call on the same input is bitwise equal
    lg2 = torch.from_numpy(x).cuda()
    rl2 = torch.empty(N, device="cuda")
    abi.echo_xent_fwd_bwd(N, V, lg2, bb, yy, rl2, None)
    assert torch.equal(lg, lg2) and torch.equal(rl, rl2)


@pytest.mark.parametrize("rows,cols,dtype", [(6400, 512, "fp32"), (33, 29, "fp32"), (1000, 2048, "bf16"),
                                             (1, 7, "fp32"),
                                             # the vectorised path (>= 1 M elements; 8 or 16 row segments)
                                             (65536, 2048, "fp32"), (4099, 8192, "fp32"), (33333, 2048, "bf16"),
                                             (3001, 1024, "bf16"), (20000, 520, "fp32")])
def test_colsum_fp64_accumulation(rows, cols, dtype, cuda_dev):
    """echo_colsum equals the fp64 column sum rounded once to fp32 (within 1 ulp), including a
    cancellation-heavy case where an fp32 sum is visibly off."""
    from paper_1805_08899_b200 import abi
    rng = np.random.default_rng(rows + cols)
    x = rng.standard_normal((rows, cols)).astype(np.float32) * 1e3
    x[-1] = -x[:-1].astype(np.float64).sum(axis=0) + rng.standard_normal(cols)   # sums ~ N(0,1): cancellation
    t = torch.from_numpy(x).cuda()
    if dtype == "bf16":
        t = t.to(torch.bfloat16)
        x = t.float().cpu().numpy()
    ref = x.astype(np.float64).sum(axis=0).astype(np.float32)
    out = torch.empty(cols, device="cuda")
    abi.echo_colsum(t, out)
    got = out.cpu().numpy()
    ulp = np.spacing(np.abs(ref))
    assert np.all(np.abs(got - ref) <= ulp), np.max(np.abs(got - ref) / ulp)
    out2 = torch.ones(cols, device="cuda")
    abi.echo_colsum(t, out2, accumulate=1)
    assert torch.allclose(out2, out + 1.0)


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("n", [1, 777, 128 * 512])
def test_tanh_bwd(storage, n, cuda_dev):
    """echo_tanh_bwd == the fp32 expression da * (1 - a*a) bitwise, and == fp64 within fp32 rounding."""
    from paper_1805_08899_b200 import abi
    g = torch.Generator(device="cuda").manual_seed(n)
    sd = torch.float32 if storage == "fp32" else torch.bfloat16
    a = torch.tanh(torch.randn(n, device="cuda", generator=g) * 2).to(sd)
    da = torch.randn(n, device="cuda", generator=g)
    out = torch.empty(n, device="cuda")
    abi.echo_tanh_bwd(a, da, out)
    af = a.float()
    assert torch.equal(out, da * (1.0 - af * af))
    ref = da.double() * (1.0 - af.double() ** 2)
    assert float((out.double() - ref).abs().max() / ref.abs().max()) < 1e-6
