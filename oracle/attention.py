"""MLP (Bahdanau) attention oracle, fp64.  TEST INFRASTRUCTURE ONLY.

PAPER.md §2 (lines 129-133): (1) a scoring function compares the query with
the encoder hidden state H_s, giving scores and weights alpha_ts; (2) the
context is the alpha-weighted average of H_s.  Fig. 7 is the
simplified scoring function: broadcast-add of the query to [T x N] then tanh.

Readings: scores / alpha are [B, Ts] (R1, the printed [B x H] is
garbled); score = v . tanh(qp + Kp_s) with qp = W_q q + b_q, Kp = W_k H_s computed
by the caller's FCs (R3); source positions s >= len_b are masked (alpha = 0,
zero gradient, R8); softmax is max-subtracted (R9).
Written with numpy broadcasting over (b, s) so it also runs at C2 sizes; each
line is one step of the definition.
Pins: tests/test_oracle_attention.py.
"""
from __future__ import annotations

import numpy as np


def _valid(B, Ts, src_len):
    if src_len is None:
        return np.ones((B, Ts), bool)
    return np.arange(Ts)[None, :] < np.asarray(src_len)[:, None]


def forward(qp, Kp, v, Hs, src_len=None):
    qp = np.asarray(qp, np.float64)
    Kp = np.asarray(Kp, np.float64)
    v = np.asarray(v, np.float64)
    Hs = np.asarray(Hs, np.float64)
    B, Ts, A = Kp.shape
    valid = _valid(B, Ts, src_len)
    E = np.tanh(qp[:, None, :] + Kp)                         # Fig. 7: broadcast-add, then tanh
    E = np.where(valid[:, :, None], E, 0.0)
    scores = np.where(valid, E @ v, -np.inf)                 # score projection, masked (R8)
    m = scores.max(axis=1, keepdims=True)
    w = np.where(valid, np.exp(scores - m), 0.0)
    alpha = w / w.sum(axis=1, keepdims=True)                 # softmax over source positions
    ctx = np.einsum("bs,bsk->bk", alpha, Hs)                 # (2) alpha-weighted average of H_s
    return {"E": E, "scores": scores, "alpha": alpha, "ctx": ctx}


def backward(qp, Kp, v, Hs, dctx, src_len=None):
    """Gradients of <dctx, ctx> w.r.t. qp, Kp, v, Hs (plus the regenerated ctx)."""
    fw = forward(qp, Kp, v, Hs, src_len)
    v = np.asarray(v, np.float64)
    Hs = np.asarray(Hs, np.float64)
    dctx = np.asarray(dctx, np.float64)
    alpha, E = fw["alpha"], fw["E"]
    dalpha = np.einsum("bk,bsk->bs", dctx, Hs)               # d ctx / d alpha_s = H_s
    ds = alpha * (dalpha - (alpha * dalpha).sum(axis=1, keepdims=True))   # softmax backward
    dE = ds[:, :, None] * v[None, None, :] * (1.0 - E * E)   # tanh' = 1 - tanh^2
    dqp = dE.sum(axis=1)                                     # broadcast-add backward: sum over s
    dKp = dE
    dv = np.einsum("bs,bsa->a", ds, E)
    dHs = alpha[:, :, None] * dctx[:, None, :]
    return {"dqp": dqp, "dKp": dKp, "dv": dv, "dHs": dHs, "ctx": fw["ctx"], "alpha": alpha, "E": E}
