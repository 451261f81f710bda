"""echo_lstm_fwd_tc: one LSTM forward step with the recurrent contraction on tcgen05 (TMEM accumulator)
and the a1 cell fused into the epilogue.  Checked against the fp64 oracle cell
(oracle.lstm.cell_forward on A = gx + h W_h^T + b with the bf16-rounded G), against the per-step path
(cuBLAS beta = 1 GEMM + echo_lstm_fwd: equal up to the GEMM's accumulation order), and STASH ==
RECOMPUTE bitwise."""
import numpy as np
import pytest
import torch

from oracle import lstm as O
from tests.gpu_util import assert_close, bits_equal, host

pytestmark = pytest.mark.gpu


def _abi():
    from paper_1805_08899_b200 import abi
    abi.load()
    return abi


def _bf(x):
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("B,H", [(128, 512), (1, 64), (37, 128), (128, 256), (100, 448)])
def test_tc_step_vs_oracle_and_per_step_path(B, H, cuda_dev):
    abi = _abi()
    assert abi.echo_lstm_fwd_tc_supported(B, H, abi.BF16)
    g = torch.Generator(device="cuda").manual_seed(B * 7 + H)
    gx = _bf(torch.randn(B, 4 * H, device="cuda", generator=g) * 0.5)
    hp = _bf(torch.randn(B, H, device="cuda", generator=g) * 0.5)
    Wh = _bf(torch.randn(4 * H, H, device="cuda", generator=g) / np.sqrt(H))
    bias = torch.randn(4 * H, device="cuda", generator=g) * 0.1
    cp = torch.randn(B, H, device="cuda", generator=g)
    res = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        d = abi.LstmDesc(B, H, abi.BF16, mode)
        gates = gx.clone()                                  # gx_t aliases gates_t (in place, as the layer does)
        c = torch.empty(B, H, device="cuda")
        tc = torch.empty(B, H, device="cuda", dtype=torch.bfloat16) if mode == abi.STASH else None
        h = torch.empty(B, H, device="cuda", dtype=torch.bfloat16)
        abi.echo_lstm_fwd_tc(d, gates, hp, Wh, bias, cp, gates, c, tc, h)
        torch.cuda.synchronize()
        res[mode] = (gates, c, h, tc)
    for k in range(3):
        assert bits_equal(res[abi.STASH][k], res[abi.RECOMPUTE][k]), k
    gates, c, h, tc = res[abi.STASH]
    # fp64 oracle on the same bf16 inputs (A = gx + h W^T + b, unrounded)
    A = host(gx) + host(hp) @ host(Wh).T + host(bias)[None, :]
    ref = O.cell_forward(A, host(cp))
    for kk, name in enumerate("ifgo"):
        assert_close(host(gates[:, kk * H:(kk + 1) * H]), ref[name], "bf16", name)
    assert_close(host(c), ref["c"], "bf16", "c")
    assert_close(host(h), ref["h"], "bf16", "h")
    # per-step path: cuBLAS beta = 1 GEMM into gx, then a1 (bias in a1)
    d = abi.LstmDesc(B, H, abi.BF16, abi.STASH)
    g2 = gx.clone()
    g2.addmm_(hp, Wh.t())
    gates2 = torch.empty_like(g2)
    c2 = torch.empty(B, H, device="cuda")
    tc2 = torch.empty(B, H, device="cuda", dtype=torch.bfloat16)
    h2 = torch.empty(B, H, device="cuda", dtype=torch.bfloat16)
    abi.echo_lstm_fwd(d, g2, None, bias, cp, gates2, c2, tc2, h2)
    torch.cuda.synchronize()
    # the same up to the rounding of G = round_bf16(gx + h W^T): the tensor-core path rounds the fp32 sum
    # once; where the two differ it is by bf16 ulps of G, propagated through the gates
    dg = (gates.float() - gates2.float()).abs()
    assert dg.max().item() <= 2.0 ** -6, dg.max().item()
    assert (c - c2).abs().max().item() <= 2e-2 * max(1.0, c2.abs().max().item())


def test_tc_step_rejects_unsupported(cuda_dev):
    abi = _abi()
    assert not abi.echo_lstm_fwd_tc_supported(129, 512, abi.BF16)
    assert not abi.echo_lstm_fwd_tc_supported(128, 512, abi.FP32)
    assert not abi.echo_lstm_fwd_tc_supported(128, 1024, abi.BF16)
    x = torch.zeros(16, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(abi.EchoError) as e:
        abi.echo_lstm_fwd_tc(abi.LstmDesc(129, 512, abi.BF16, abi.RECOMPUTE), x, x, x, x.float(), x.float(), x, x.float(),
                             None, x)
    assert e.value.status == abi.ECHO_ERR_UNSUPPORTED
