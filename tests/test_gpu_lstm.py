"""GPU parity of the LSTM kernels a1/a2/a3 (through the C ABI) against the fp64 oracle,
and STASH == RECOMPUTE bit-identity."""
import numpy as np
import pytest
import torch

from oracle import lstm as O
from synth.data import lstm_layer_inputs, lstm_cell_inputs
from tests.gpu_util import dev, host, assert_close, bits_equal

pytestmark = pytest.mark.gpu

STORAGES = ["fp32", "bf16"]


@pytest.fixture(autouse=True)
def _strict_fp32():
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.allow_tf32 = False


def _abi():
    from paper_1805_08899_b200 import abi
    abi.load()
    return abi


@pytest.mark.parametrize("storage", STORAGES)
@pytest.mark.parametrize("mode", ["stash", "recompute"])
@pytest.mark.parametrize("B,H", [(3, 16), (5, 40), (128, 512), (24576, 512)])
def test_cell_fwd_bwd_step(storage, mode, B, H, cuda_dev):
    """a1 + a3 on one step vs oracle cell_forward / cell_backward (A given); B = 24576 is C5's
    per-step launch configuration (every row compared)."""
    abi = _abi()
    d = lstm_cell_inputs(11, B, H, storage)
    m = abi.STASH if mode == "stash" else abi.RECOMPUTE
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    desc = abi.LstmDesc(B, H, dt, m)
    A = dev(d["A"], storage)
    cp = dev(d["c_prev"], dtype=torch.float32)
    gates = torch.empty_like(A)
    c = torch.empty(B, H, device="cuda")
    tc = torch.empty(B, H, device="cuda", dtype=A.dtype) if m == abi.STASH else None
    h = torch.empty(B, H, device="cuda", dtype=A.dtype)
    abi.echo_lstm_fwd(desc, A, None, None, cp, gates, c, tc, h)
    ref = O.cell_forward(np.asarray(d["A"], np.float64), np.asarray(d["c_prev"], np.float64))
    Hh = H
    g = host(gates)
    for k, name in enumerate("ifgo"):
        assert_close(g[:, k * Hh:(k + 1) * Hh], ref[name], storage, name)
    assert_close(host(c), ref["c"], storage, "c")
    assert_close(host(h), ref["h"], storage, "h")
    dh = dev(d["dh"], dtype=torch.float32)
    dc = dev(d["dc"], dtype=torch.float32)
    dA = torch.empty_like(A)
    hreg = torch.empty_like(h) if m == abi.RECOMPUTE else None
    if m == abi.STASH:
        abi.echo_lstm_bwd(desc, gates, cp, None, tc, dh, dc, dA, None)
    else:
        abi.echo_lstm_bwd(desc, gates, cp, c, None, dh, dc, dA, hreg)
        assert bits_equal(hreg, h)          # regenerated h_t bit-identical to the forward's
    rdA, rdc = O.cell_backward(np.asarray(d["A"], np.float64), np.asarray(d["c_prev"], np.float64),
                               np.asarray(d["dh"], np.float64), np.asarray(d["dc"], np.float64))
    assert_close(host(dA), rdA, storage, "dA")
    assert_close(host(dc), rdc, storage, "dc")


@pytest.mark.parametrize("storage", STORAGES)
@pytest.mark.parametrize("T,B,I,H", [(4, 2, 16, 16), (7, 3, 24, 40), (50, 128, 512, 512)])
def test_layer_parity_and_bit_identity(storage, T, B, I, H, cuda_dev):
    """Full layer forward + BPTT in both modes vs the oracle; STASH and RECOMPUTE grads bitwise equal."""
    abi = _abi()
    from paper_1805_08899_b200.lstm import LSTMLayer
    d = lstm_layer_inputs(21, T, B, I, H, storage)
    ref = O.layer_backward(*(np.asarray(d[k], np.float64) for k in ("X", "Wx", "Wh", "b", "h0", "c0")),
                           dH=np.asarray(d["dH"], np.float64), dcT=np.asarray(d["dcT"], np.float64))
    outs = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        L = LSTMLayer(T, B, H, abi.FP32 if storage == "fp32" else abi.BF16, mode)
        X, Wx, Wh = dev(d["X"], storage), dev(d["Wx"], storage), dev(d["Wh"], storage)
        b = dev(d["b"], dtype=torch.float32)
        h0, c0 = dev(d["h0"], storage), dev(d["c0"], dtype=torch.float32)
        Hout = L.forward_seq(X, Wx, Wh, b, h0, c0).clone()
        cT = L.c_final().clone()
        g = L.backward_seq(X, Wx, Wh, dev(d["dH"], dtype=torch.float32), dcT=dev(d["dcT"], dtype=torch.float32))
        outs[mode] = (Hout, cT, g)
        assert_close(host(Hout), ref["fw"]["H"], storage, "H")
        assert_close(host(cT), ref["fw"]["cT"], storage, "cT")
        for k in ("dX", "dWx", "dWh", "db", "dh0", "dc0"):
            assert_close(host(g[k]), ref[k], storage, k)
    s, r = outs[abi.STASH], outs[abi.RECOMPUTE]
    assert bits_equal(s[0], r[0]) and bits_equal(s[1], r[1])
    for k in s[2]:
        assert bits_equal(s[2][k], r[2][k]), f"STASH vs RECOMPUTE differ in {k}"


@pytest.mark.parametrize("storage", STORAGES)
def test_cscan_regenerates_h_bitwise(storage, cuda_dev):
    abi = _abi()
    from paper_1805_08899_b200.lstm import LSTMLayer
    T, B, I, H = 9, 5, 16, 40
    d = lstm_layer_inputs(4, T, B, I, H, storage)
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    S = LSTMLayer(T, B, H, dt, abi.STASH)
    S.forward_seq(dev(d["X"], storage), dev(d["Wx"], storage), dev(d["Wh"], storage), dev(d["b"], dtype=torch.float32),
                  dev(d["h0"], storage), dev(d["c0"], dtype=torch.float32))
    cws = torch.empty(T, B, H, device="cuda")
    hws = torch.empty_like(S.h)
    abi.echo_lstm_cscan(abi.LstmDesc(B, H, dt, abi.RECOMPUTE), T, S.gates, S.c0, cws, hws)
    assert bits_equal(cws[: T - 1], S.c[: T - 1]) and bits_equal(hws, S.h)


def test_cscan_matches_forward_c_bitwise(cuda_dev):
    """a2 regenerates exactly the c_t the forward produced (same device function)."""
    abi = _abi()
    from paper_1805_08899_b200.lstm import LSTMLayer
    T, B, I, H = 33, 9, 8, 24
    d = lstm_layer_inputs(3, T, B, I, H)
    S = LSTMLayer(T, B, H, abi.FP32, abi.STASH)
    S.forward_seq(dev(d["X"]), dev(d["Wx"]), dev(d["Wh"]), dev(d["b"]), dev(d["h0"]), dev(d["c0"]))
    cws = torch.empty(T, B, H, device="cuda")
    hws = torch.empty(T, B, H, device="cuda")
    abi.echo_lstm_cscan(abi.LstmDesc(B, H, abi.FP32, abi.RECOMPUTE), T, S.gates, S.c0, cws, hws)
    assert bits_equal(cws, S.c)
    assert bits_equal(hws, S.h)          # mirrored layer outputs regenerate bit-identically


def test_validation_errors(cuda_dev):
    abi = _abi()
    B, H = 2, 12   # H not a multiple of 8
    t = torch.empty(B, 4 * H, device="cuda")
    with pytest.raises(abi.EchoError) as e:
        abi.echo_lstm_fwd(abi.LstmDesc(B, H, abi.FP32, abi.RECOMPUTE), t, None, None, t, t, t, None, t)
    assert e.value.status == abi.ECHO_ERR_INVALID
    B, H = 2, 16
    t = torch.empty(B, 4 * H, device="cuda")
    c = torch.empty(B, H, device="cuda")
    with pytest.raises(abi.EchoError):   # STASH requires tc
        abi.echo_lstm_fwd(abi.LstmDesc(B, H, abi.FP32, abi.STASH), t, None, None, c, t, c.clone(), None, c.clone())
    with pytest.raises(abi.EchoError):   # misaligned pointer
        abi.echo_lstm_fwd(abi.LstmDesc(B, H, abi.FP32, abi.RECOMPUTE), t.view(-1)[1:].data_ptr(), None, None, c, t,
                          c.clone(), None, c.clone())
