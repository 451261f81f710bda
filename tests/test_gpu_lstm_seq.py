"""Fused persistent LSTM forward (echo_lstm_seq_fwd, a1 over the recurrence) vs the fp64 oracle
layer, vs the per-step path (GEMM + echo_lstm_fwd), STASH == RECOMPUTE
bitwise, chunked launches == one launch bitwise, and the reverse direction."""
import numpy as np
import pytest
import torch

from oracle import lstm as O
from synth.data import lstm_layer_inputs
from tests.gpu_util import dev, host, assert_close, bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _strict_fp32():
    torch.backends.cuda.matmul.allow_tf32 = False


def _layer(abi, d, storage, mode, reverse, chunks):
    from paper_1805_08899_b200.lstm import LSTMLayer
    T, B, _ = d["X"].shape
    H = d["Wh"].shape[1]
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    L = LSTMLayer(T, B, H, dt, mode, "cuda", reverse=reverse)
    X, Wx, Wh = dev(d["X"], storage), dev(d["Wx"], storage), dev(d["Wh"], storage)
    b = dev(d["b"], dtype=torch.float32)
    h0, c0 = dev(d["h0"], storage), dev(d["c0"], dtype=torch.float32)
    L.h0, L.c0 = h0, c0
    GX = torch.empty(T, B, 4 * H, dtype=X.dtype, device="cuda") if reverse else L.gates
    torch.mm(X.reshape(T * B, -1), Wx.t(), out=GX.view(T * B, 4 * H))
    bounds = [(T * i) // chunks for i in range(chunks + 1)]
    for k0, k1 in zip(bounds[:-1], bounds[1:]):
        L.fused_steps(k0, k1, GX, Wh, b)
    torch.cuda.synchronize()
    return L


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
@pytest.mark.parametrize("T,B,I,H", [(7, 32, 24, 64), (5, 64, 40, 128), (4, 128, 64, 512), (3, 32, 48, 800)])
@pytest.mark.parametrize("reverse", [False, True])
def test_seq_fwd_vs_oracle_and_modes(storage, T, B, I, H, reverse, cuda_dev):
    from paper_1805_08899_b200 import abi
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    if not abi.echo_lstm_seq_supported(B, H, dt):
        pytest.skip("no co-resident tile on this device")
    d = lstm_layer_inputs(5 + H, T, B, I, H, storage)
    X = d["X"][::-1] if reverse else d["X"]
    ref = O.layer_forward(X, d["Wx"], d["Wh"], d["b"], d["h0"], d["c0"])
    outs = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        L = _layer(abi, d, storage, mode, reverse, 1)
        Hg = host(L.h)
        Hr = ref["H"][::-1] if reverse else ref["H"]              # outputs by time
        assert_close(Hg, Hr, storage, "h")
        outs[mode] = L
    s, r = outs[abi.STASH], outs[abi.RECOMPUTE]
    assert_close(host(s.c), ref["C"], storage, "c")
    assert bits_equal(s.gates, r.gates) and bits_equal(s.h, r.h)
    assert bits_equal(s.c[T - 1], r.c_final())
    # chunked launches (the encoder wavefront) == one launch, bitwise
    L3 = _layer(abi, d, storage, abi.RECOMPUTE, reverse, 3 if T >= 3 else 1)
    assert bits_equal(L3.gates, r.gates) and bits_equal(L3.h, r.h)


def test_seq_fwd_close_to_per_step_path(cuda_dev):
    """C2 encoder shapes: the fused launch agrees with the per-step GEMM + a1 path to fp32 rounding."""
    import os
    from paper_1805_08899_b200 import abi
    from paper_1805_08899_b200.lstm import LSTMLayer
    T, B, I, H = 10, 128, 512, 512
    if not abi.echo_lstm_seq_supported(B, H, abi.FP32):
        pytest.skip("no co-resident tile on this device")
    d = lstm_layer_inputs(3, T, B, I, H, "fp32")
    X, Wx, Wh = dev(d["X"]), dev(d["Wx"]), dev(d["Wh"])
    b, h0, c0 = dev(d["b"]), dev(d["h0"]), dev(d["c0"])
    res = {}
    for flag in ("0", "1"):
        os.environ["ECHO_LSTM_FUSED"] = flag
        L = LSTMLayer(T, B, H, abi.FP32, abi.RECOMPUTE, "cuda")
        assert L.fused_ok() == (flag == "1")
        L.forward_seq(X, Wx, Wh, b, h0, c0)
        res[flag] = L.h.clone()
    os.environ.pop("ECHO_LSTM_FUSED")
    assert_close(host(res["1"]), host(res["0"]), "fp32", "fused vs per-step")
