"""LSTM oracle (fp64, explicit loops over t).  TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2 (lines 101-112, Fig. 1): each cell takes i_t and h_{t-1}
through a fully-connected layer Y = X W^T + b with W: [4H x H] (Eq. 1,
PAPER.md:104-106), then the non-linear block f ("slicing and element-wise
operations") produces h_t and c_t, both [B x H].

Readings: gate order i|f|g|o as contiguous H-blocks (R4); one bias
b = b_ih + b_hh per layer (R5); h0, c0 are caller inputs (R6).
Pins: tests/test_oracle_lstm.py (central FD, zero-weight closed form,
saturation closed form, torch.nn.LSTM fp64 cross-check).
"""
from __future__ import annotations

import numpy as np


def sigmoid(x):
    with np.errstate(over="ignore"):          # exp(+large) = inf gives exactly 0, as intended
        return 1.0 / (1.0 + np.exp(-x))


def cell_forward(A, c_prev):
    """Non-linear block f of one cell.  A = x W_x^T + h W_h^T + b, [B, 4H]."""
    A = np.asarray(A, np.float64)
    H = A.shape[1] // 4
    i = sigmoid(A[:, 0 * H:1 * H])
    f = sigmoid(A[:, 1 * H:2 * H])
    g = np.tanh(A[:, 2 * H:3 * H])
    o = sigmoid(A[:, 3 * H:4 * H])
    c = f * c_prev + i * g
    tc = np.tanh(c)
    h = o * tc
    return {"i": i, "f": f, "g": g, "o": o, "c": c, "tc": tc, "h": h}


def cell_backward(A, c_prev, dh, dc_next):
    """Gradient of the non-linear block: returns dA [B,4H] and dc_prev [B,H].

    Chain rule on h = o*tanh(c), c = f*c_prev + i*g with sigma' = s(1-s),
    tanh' = 1 - tanh^2 (PAPER.md:195 for the tanh derivative).
    """
    s = cell_forward(A, c_prev)
    i, f, g, o, tc = s["i"], s["f"], s["g"], s["o"], s["tc"]
    do = dh * tc
    dc = dc_next + dh * o * (1.0 - tc * tc)
    di = dc * g
    dg = dc * i
    df = dc * c_prev
    dc_prev = dc * f
    dA = np.concatenate([di * i * (1.0 - i), df * f * (1.0 - f), dg * (1.0 - g * g), do * o * (1.0 - o)], axis=1)
    return dA, dc_prev


def layer_forward(X, Wx, Wh, b, h0, c0):
    """Unrolled LSTM layer over T steps (Fig. 1 left).  X [T,B,I]."""
    X = np.asarray(X, np.float64)
    T = X.shape[0]
    h, c = np.asarray(h0, np.float64), np.asarray(c0, np.float64)
    Hs, Cs, As = [], [], []
    for t in range(T):
        A = X[t] @ np.asarray(Wx, np.float64).T + h @ np.asarray(Wh, np.float64).T + np.asarray(b, np.float64)
        s = cell_forward(A, c)
        h, c = s["h"], s["c"]
        As.append(A)
        Hs.append(h)
        Cs.append(c)
    return {"H": np.stack(Hs), "C": np.stack(Cs), "A": np.stack(As), "hT": h, "cT": c}


def layer_backward(X, Wx, Wh, b, h0, c0, dH, dhT=None, dcT=None):
    """BPTT through one layer.  dH [T,B,H] is dLoss/dh_t from above (all t).

    Returns dX, dWx, dWh, db, dh0, dc0 and the per-step dA [T,B,4H].
    FC gradients follow Eq. 2: dX = dY W, dW = dY^T X.
    """
    X = np.asarray(X, np.float64)
    Wx = np.asarray(Wx, np.float64)
    Wh = np.asarray(Wh, np.float64)
    fw = layer_forward(X, Wx, Wh, b, h0, c0)
    T, B, _ = X.shape
    H = Wh.shape[1]
    h0 = np.asarray(h0, np.float64)
    c0 = np.asarray(c0, np.float64)
    dX = np.zeros_like(X)
    dWx = np.zeros_like(Wx)
    dWh = np.zeros_like(Wh)
    db = np.zeros(4 * H)
    dA_all = np.zeros((T, B, 4 * H))
    dh_rec = np.zeros((B, H)) if dhT is None else np.asarray(dhT, np.float64).copy()
    dc = np.zeros((B, H)) if dcT is None else np.asarray(dcT, np.float64).copy()
    for t in reversed(range(T)):
        c_prev = c0 if t == 0 else fw["C"][t - 1]
        h_prev = h0 if t == 0 else fw["H"][t - 1]
        dh = np.asarray(dH[t], np.float64) + dh_rec
        dA, dc = cell_backward(fw["A"][t], c_prev, dh, dc)
        dA_all[t] = dA
        dh_rec = dA @ Wh
        dWh += dA.T @ h_prev
        dWx += dA.T @ X[t]
        db += dA.sum(axis=0)
        dX[t] = dA @ Wx
    return {"dX": dX, "dWx": dWx, "dWh": dWh, "db": db, "dh0": dh_rec, "dc0": dc, "dA": dA_all, "fw": fw}
