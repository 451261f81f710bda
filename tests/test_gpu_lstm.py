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
    if m == abi.STASH:                      # one step: T = 1, t = 0, c_0 = c_prev
        abi.echo_lstm_bwd_recompute(desc, 1, 0, 0, gates, cp, None, tc, dh, dc, dA, None, None)
    else:                                   # the a2 workspace holds c_1 = c
        abi.echo_lstm_bwd_recompute(desc, 1, 0, 0, gates, cp, None, None, dh, dc, dA, hreg, c)
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


@pytest.mark.parametrize("storage", STORAGES)
def test_bwd_recompute_regen_flag_and_ws_query(storage, cuda_dev):
    """echo_lstm_bwd_recompute with ECHO_BWD_REGEN_C on the first backward call (the a2 prologue
    inside the entry point, workspace sized by the two-call query) == the layer driver's separate
    scan + per-step calls, bitwise; the STASH calls through the same entry point agree too."""
    abi = _abi()
    from paper_1805_08899_b200.lstm import LSTMLayer
    T, B, I, H = 12, 6, 16, 40
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    d = lstm_layer_inputs(8, T, B, I, H, storage)
    ins = lambda: (dev(d["X"], storage), dev(d["Wx"], storage), dev(d["Wh"], storage), dev(d["b"], dtype=torch.float32),
                   dev(d["h0"], storage), dev(d["c0"], dtype=torch.float32))
    dH = dev(d["dH"], dtype=torch.float32)
    res = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        L = LSTMLayer(T, B, H, dt, mode)
        L.forward_seq(*ins())
        desc = abi.LstmDesc(B, H, dt, mode)
        nb = abi.echo_lstm_bwd_ws_bytes(desc, T)
        assert nb == (T * B * H * 4 if mode == abi.RECOMPUTE else 0)
        ws = torch.full((max(nb, 4) // 4,), float("nan"), device="cuda")
        gates = L.gates.clone()
        dc = torch.zeros(B, H, device="cuda")
        hreg = torch.empty(T, B, H, device="cuda", dtype=L.sd)
        for t in reversed(range(T)):
            if mode == abi.RECOMPUTE:
                abi.echo_lstm_bwd_recompute(desc, T, t, abi.ECHO_BWD_REGEN_C if t == T - 1 else 0, gates, L.c0, None,
                                            None, dH[t], dc, gates[t], hreg[t], ws, nb)
            else:
                abi.echo_lstm_bwd_recompute(desc, T, t, 0, gates, L.c0, L.c, L.tc, dH[t], dc, gates[t], None, None)
        res[mode] = (gates, dc)
        if mode == abi.RECOMPUTE:
            assert bits_equal(hreg, L.h)
        # the driver's path (separate scan + per-step calls) on the same stashed gates
        L.prepare_backward()
        dc2 = torch.zeros(B, H, device="cuda")
        for t in reversed(range(T)):
            L.bwd_step(t, dH[t], dc2)
        assert bits_equal(L.gates, gates) and bits_equal(dc2, dc)
    assert bits_equal(res[abi.STASH][0], res[abi.RECOMPUTE][0]) and bits_equal(res[abi.STASH][1], res[abi.RECOMPUTE][1])
    # validation: t out of range, flag in STASH mode, workspace too small
    desc = abi.LstmDesc(B, H, dt, abi.RECOMPUTE)
    g = torch.empty(T, B, 4 * H, device="cuda", dtype=L.sd)
    c0 = torch.zeros(B, H, device="cuda")
    for args, st in (((T, T, 0), abi.ECHO_ERR_INVALID), ((T, 0, 4), abi.ECHO_ERR_INVALID)):
        with pytest.raises(abi.EchoError) as e:
            abi.echo_lstm_bwd_recompute(desc, *args, g, c0, None, None, c0, c0.clone(), g[0], None, ws)
        assert e.value.status == st
    with pytest.raises(abi.EchoError) as e:
        abi.echo_lstm_bwd_recompute(desc, T, 0, 0, g, c0, None, None, c0, c0.clone(), g[0], None, ws, 16)
    assert e.value.status == abi.ECHO_ERR_CAPACITY
    with pytest.raises(abi.EchoError) as e:
        abi.echo_lstm_bwd_recompute(abi.LstmDesc(B, H, dt, abi.STASH), T, 0, abi.ECHO_BWD_REGEN_C, g, c0, g, g, c0,
                                    c0.clone(), g[0], None, None)
    assert e.value.status == abi.ECHO_ERR_INVALID


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


@pytest.mark.parametrize("storage", STORAGES)
@pytest.mark.parametrize("n_parts", [1, 2, 3])
@pytest.mark.parametrize("B,H", [(3, 16), (128, 512)])
def test_mirror_parts_kernels(storage, n_parts, B, H, cuda_dev):
    """Mirror-plan kernels (echo_lstm_*_parts): A = ((P0 + P1) + P2) + b in fp32; forward, scan and
    backward vs the oracle cell on that A; fwd_parts with two parts == a1 with (gx, gh, bias)
    bitwise; the scan's c == the forward's c bitwise; bwd_parts == a3 (RECOMPUTE) on a1's gates."""
    abi = _abi()
    rng = np.random.default_rng(B * 10 + n_parts)
    sd = torch.float32 if storage == "fp32" else torch.bfloat16
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    desc = abi.LstmDesc(B, H, dt, abi.RECOMPUTE)
    T = 3
    parts = torch.from_numpy(rng.standard_normal((n_parts, T, B, 4 * H)).astype(np.float32) * 0.7).cuda().to(sd)
    bias = torch.from_numpy(rng.standard_normal(4 * H).astype(np.float32) * 0.3).cuda()
    c0 = torch.from_numpy(rng.standard_normal((B, H)).astype(np.float32)).cuda()
    ps = T * B * 4 * H
    A = parts[0].float()
    for q in range(1, n_parts):
        A = A + parts[q].float()
    A = A + bias
    # forward over T steps
    c = [c0]
    h = torch.empty(T, B, H, dtype=sd, device="cuda")
    for t in range(T):
        c.append(torch.empty(B, H, device="cuda"))
        abi.echo_lstm_fwd_parts(desc, n_parts, parts[0][t], ps, bias, c[t], c[t + 1], h[t])
    for t in range(T):
        ref = O.cell_forward(host(A[t]), host(c[t]))
        assert_close(host(c[t + 1]), ref["c"], storage, "c")
        assert_close(host(h[t]), ref["h"], storage, "h")
    if n_parts == 2:                                   # same arithmetic as a1 with gx, gh, bias
        g1 = torch.empty(B, 4 * H, dtype=sd, device="cuda")
        c1 = torch.empty(B, H, device="cuda")
        h1 = torch.empty(B, H, dtype=sd, device="cuda")
        abi.echo_lstm_fwd(desc, parts[0][0], parts[1][0], bias, c0, g1, c1, None, h1)
        assert bits_equal(c1, c[1]) and bits_equal(h1, h[0])
    cws = torch.empty(T, B, H, device="cuda")
    abi.echo_lstm_cscan_parts(desc, T, n_parts, parts[0][0], ps, B * 4 * H, bias, c0, cws)
    for t in range(T):
        assert bits_equal(cws[t], c[t + 1])
    cws_r = torch.empty(T, B, H, device="cuda")            # reverse walk (negative step stride)
    abi.echo_lstm_cscan_parts(desc, T, n_parts, parts[0][T - 1], ps, -B * 4 * H, bias, c0, cws_r)
    cr = c0
    for k in range(T):
        ref = O.cell_forward(host(A[T - 1 - k]), host(cr))
        assert_close(host(cws_r[k]), ref["c"], storage, "c reverse")
        cr = cws_r[k]
    # backward of the last step vs the oracle, and (fp32) vs a3 on a1's gates bitwise
    dh = torch.from_numpy(rng.standard_normal((B, H)).astype(np.float32)).cuda()
    dc_in = torch.from_numpy(rng.standard_normal((B, H)).astype(np.float32)).cuda()
    dc = dc_in.clone()
    dA = torch.empty(B, 4 * H, dtype=sd, device="cuda")
    abi.echo_lstm_bwd_parts(desc, n_parts, parts[0][T - 1], ps, bias, c[T - 1], c[T], dh, dc, dA)
    rdA, rdc = O.cell_backward(host(A[T - 1]), host(c[T - 1]), host(dh), host(dc_in))
    assert_close(host(dA), rdA, storage, "dA")
    assert_close(host(dc), rdc, storage, "dc")
    if storage == "fp32":                                 # a1 on the fp32 A itself: the same gates
        gates = torch.empty(B, 4 * H, device="cuda")
        cc = torch.empty(B, H, device="cuda")
        hh = torch.empty(B, H, device="cuda")
        abi.echo_lstm_fwd(desc, A[T - 1].contiguous(), None, None, c[T - 1], gates, cc, None, hh)
        dc2 = dc_in.clone()
        dA2 = torch.empty_like(dA)
        abi.echo_lstm_bwd_recompute(abi.LstmDesc(B, H, abi.FP32, abi.RECOMPUTE), 1, 0, 0, gates, c[T - 1], None, None,
                                    dh, dc2, dA2, None, c[T])
        assert bits_equal(dA, dA2) and bits_equal(dc, dc2)
