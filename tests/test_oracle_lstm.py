"""Pins for oracle/lstm.py against things other than itself (SURVEY.md §8(c) pins O1)."""
import numpy as np
import pytest
import torch

from oracle import lstm as O
from synth.data import lstm_layer_inputs


def _loss(X, Wx, Wh, b, h0, c0, R, RT, RC):
    fw = O.layer_forward(X, Wx, Wh, b, h0, c0)
    return (fw["H"] * R).sum() + (fw["hT"] * RT).sum() + (fw["cT"] * RC).sum()


def test_fd_all_gradients_c1():
    """Central finite differences (eps=1e-6) of a random linear functional (pin: FD)."""
    d = lstm_layer_inputs(1, T=4, B=2, I=16, H=16)
    g = np.random.default_rng(7)
    R = g.standard_normal((4, 2, 16))
    RT = g.standard_normal((2, 16))
    RC = g.standard_normal((2, 16))
    args = {k: np.asarray(d[k], np.float64) for k in ("X", "Wx", "Wh", "b", "h0", "c0")}
    bw = O.layer_backward(args["X"], args["Wx"], args["Wh"], args["b"], args["h0"], args["c0"], R, dhT=RT, dcT=RC)
    names = {"X": "dX", "Wx": "dWx", "Wh": "dWh", "b": "db", "h0": "dh0", "c0": "dc0"}
    eps = 1e-6
    for k, gk in names.items():
        num = np.zeros_like(args[k])
        it = np.nditer(args[k], flags=["multi_index"])
        for _ in it:
            idx = it.multi_index
            a_p = {kk: v.copy() for kk, v in args.items()}
            a_m = {kk: v.copy() for kk, v in args.items()}
            a_p[k][idx] += eps
            a_m[k][idx] -= eps
            num[idx] = (_loss(**a_p, R=R, RT=RT, RC=RC) - _loss(**a_m, R=R, RT=RT, RC=RC)) / (2 * eps)
        err = np.abs(num - bw[gk]).max() / max(np.abs(num).max(), 1e-30)
        assert err < 1e-6, (k, err)


def test_zero_weights_closed_form():
    """W=0, b=0 => i=f=o=1/2, g=0 => c_t = c0/2^t, h_t = tanh(c0/2^t)/2 (exact in fp64)."""
    T, B, H, I = 5, 3, 4, 6
    c0 = np.random.default_rng(0).standard_normal((B, H))
    fw = O.layer_forward(np.ones((T, B, I)), np.zeros((4 * H, I)), np.zeros((4 * H, H)), np.zeros(4 * H),
                         np.ones((B, H)), c0)
    for t in range(T):
        ct = c0 / 2.0 ** (t + 1)
        assert np.array_equal(fw["C"][t], ct)
        assert np.array_equal(fw["H"][t], 0.5 * np.tanh(ct))


def test_saturated_gates_closed_form():
    """b_i = -1000, b_f = +40: i = 0 and f = 1 exactly in fp64 => c_t = c0, dA_i = dA_f = 0."""
    T, B, H, I = 3, 2, 4, 5
    g = np.random.default_rng(3)
    b = g.standard_normal(4 * H) * 0.1
    b[:H] = -1000.0
    b[H:2 * H] = 40.0
    Wx = g.standard_normal((4 * H, I)) * 0.01
    Wh = g.standard_normal((4 * H, H)) * 0.01
    c0 = g.standard_normal((B, H))
    X = g.standard_normal((T, B, I))
    fw = O.layer_forward(X, Wx, Wh, b, np.zeros((B, H)), c0)
    for t in range(T):
        assert np.array_equal(fw["C"][t], c0)
    bw = O.layer_backward(X, Wx, Wh, b, np.zeros((B, H)), c0, g.standard_normal((T, B, H)))
    assert np.all(bw["dA"][:, :, :2 * H] == 0.0)


def test_torch_nn_lstm_fp64_crosscheck():
    """torch.nn.LSTM (gate order i,f,g,o; b = b_ih + b_hh) in fp64: forward and autograd backward."""
    d = lstm_layer_inputs(5, T=6, B=3, I=7, H=5)
    args = {k: np.asarray(d[k], np.float64) for k in ("X", "Wx", "Wh", "b", "h0", "c0")}
    m = torch.nn.LSTM(7, 5).double()
    with torch.no_grad():
        m.weight_ih_l0.copy_(torch.from_numpy(args["Wx"]))
        m.weight_hh_l0.copy_(torch.from_numpy(args["Wh"]))
        m.bias_ih_l0.copy_(torch.from_numpy(args["b"]) * 0.25)
        m.bias_hh_l0.copy_(torch.from_numpy(args["b"]) * 0.75)
    X = torch.from_numpy(args["X"]).requires_grad_(True)
    h0 = torch.from_numpy(args["h0"])[None].requires_grad_(True)
    c0 = torch.from_numpy(args["c0"])[None].requires_grad_(True)
    Y, (hT, cT) = m(X, (h0, c0))
    fw = O.layer_forward(**args)
    assert np.abs(Y.detach().numpy() - fw["H"]).max() < 1e-12
    assert np.abs(cT.detach().numpy()[0] - fw["cT"]).max() < 1e-12
    dH = np.asarray(d["dH"], np.float64)
    (Y * torch.from_numpy(dH)).sum().backward()
    bw = O.layer_backward(**args, dH=dH)
    assert np.abs(X.grad.numpy() - bw["dX"]).max() < 1e-12
    assert np.abs(m.weight_ih_l0.grad.numpy() - bw["dWx"]).max() < 1e-12
    assert np.abs(m.weight_hh_l0.grad.numpy() - bw["dWh"]).max() < 1e-12
    assert np.abs(m.bias_ih_l0.grad.numpy() - bw["db"]).max() < 1e-12
    assert np.abs(h0.grad.numpy()[0] - bw["dh0"]).max() < 1e-12
    assert np.abs(c0.grad.numpy()[0] - bw["dc0"]).max() < 1e-12


def test_hand_computed_single_cell():
    """T=1, B=H=1: A = [0, ln 3, atanh(1/2), 0] => i=1/2, f=3/4, g=1/2, o=1/2; c0=2 => c=3/2+1/4."""
    A = np.array([[0.0, np.log(3.0), np.arctanh(0.5), 0.0]])
    s = O.cell_forward(A, np.array([[2.0]]))
    assert abs(s["i"][0, 0] - 0.5) < 1e-15 and abs(s["f"][0, 0] - 0.75) < 1e-15
    assert abs(s["g"][0, 0] - 0.5) < 1e-15 and abs(s["o"][0, 0] - 0.5) < 1e-15
    assert abs(s["c"][0, 0] - 1.75) < 1e-15
    assert abs(s["h"][0, 0] - 0.5 * np.tanh(1.75)) < 1e-15
