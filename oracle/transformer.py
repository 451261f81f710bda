"""Transformer attention-block stack oracle, fp64.  TEST INFRASTRUCTURE ONLY.

PAPER.md §6.3.2 (line 1002): Echo recomputes the attention scores / softmax of the Transformer
and binarizes the dropout feature maps.  Block k (reading R27):
  Q = x Wq^T, K = x Wk^T, V = x Wv^T          (FCs, Eq. 1)
  per head h: P = softmax(scale * Q_h K_h^T), P_d = P * m / (1 - p)   (m: Philox keep-mask, R19)
  O_h = P_d V_h ;  y = concat_h(O_h) Wo^T + x   (residual)
Loss = mean over the B*L positions of y_final . r.
Pins: tests/test_oracle_transformer.py (FD; p = 0 with one block and one head reduces to the
plain attention formula written with torch.softmax; heads = 4, p = 0.1, two blocks against a torch
fp64 model that takes each head as a column slice and applies the same keep-mask -- forward and
every gradient to 1e-12).
"""
from __future__ import annotations

import numpy as np

from .dot_softmax import dropout_keep_mask


def _heads(X, B, L, H):
    d = X.shape[-1]
    return X.reshape(B, L, H, d // H).transpose(0, 2, 1, 3)          # [B, H, L, dh]


def _merge(Xh):
    B, H, L, dh = Xh.shape
    return Xh.transpose(0, 2, 1, 3).reshape(B, L, H * dh)


def masks(cfg, seeds):
    n = cfg.B * cfg.heads * cfg.L * cfg.L
    return [dropout_keep_mask(s, 0, n, cfg.dropout_p).reshape(cfg.B, cfg.heads, cfg.L, cfg.L) for s in seeds]


def step(params, batch, cfg, keep=None, need_grads=True):
    P = {k: np.asarray(v, np.float64) for k, v in params.items()}
    B, L, H, p = cfg.B, cfg.L, cfg.heads, cfg.dropout_p
    dh = cfg.d_model // H
    scale = 1.0 / np.sqrt(dh)
    if keep is None:
        keep = masks(cfg, batch["seeds"])
    x = np.asarray(batch["x"], np.float64)
    cache = []
    for k in range(cfg.blocks):
        Q, K, V = x @ P[f"b{k}.Wq"].T, x @ P[f"b{k}.Wk"].T, x @ P[f"b{k}.Wv"].T
        Qh, Kh, Vh = _heads(Q, B, L, H), _heads(K, B, L, H), _heads(V, B, L, H)
        S = Qh @ Kh.transpose(0, 1, 3, 2)
        Z = scale * S
        Pr = np.exp(Z - Z.max(axis=-1, keepdims=True))
        Pr /= Pr.sum(axis=-1, keepdims=True)
        Pd = Pr * keep[k] / (1.0 - p)
        O = _merge(Pd @ Vh)
        y = O @ P[f"b{k}.Wo"].T + x
        cache.append((x, Qh, Kh, Vh, Pr, O))
        x = y
    N = B * L
    loss = float((x @ P["out.r"]).sum() / N)
    out = {"loss": loss, "y": x}
    if not need_grads:
        return out
    G = {k: np.zeros_like(v) for k, v in P.items()}
    G["out.r"] = x.reshape(N, -1).sum(axis=0) / N
    dy = np.broadcast_to(P["out.r"] / N, x.shape).copy()
    for k in reversed(range(cfg.blocks)):
        xin, Qh, Kh, Vh, Pr, O = cache[k]
        G[f"b{k}.Wo"] = dy.reshape(N, -1).T @ O.reshape(N, -1)
        dO = _heads(dy @ P[f"b{k}.Wo"], B, L, H)
        Pd = Pr * keep[k] / (1.0 - p)
        dVh = Pd.transpose(0, 1, 3, 2) @ dO
        dPd = dO @ Vh.transpose(0, 1, 3, 2)
        dP = dPd * keep[k] / (1.0 - p)
        dS = scale * Pr * (dP - (Pr * dP).sum(axis=-1, keepdims=True))   # softmax backward
        dQh = dS @ Kh
        dKh = dS.transpose(0, 1, 3, 2) @ Qh
        dQ, dK, dV = _merge(dQh), _merge(dKh), _merge(dVh)
        G[f"b{k}.Wq"] = dQ.reshape(N, -1).T @ xin.reshape(N, -1)
        G[f"b{k}.Wk"] = dK.reshape(N, -1).T @ xin.reshape(N, -1)
        G[f"b{k}.Wv"] = dV.reshape(N, -1).T @ xin.reshape(N, -1)
        dy = dy + dQ @ P[f"b{k}.Wq"] + dK @ P[f"b{k}.Wk"] + dV @ P[f"b{k}.Wv"]
    out["grads"] = G
    out["dx"] = dy
    return out
