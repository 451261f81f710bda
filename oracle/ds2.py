"""DeepSpeech2-shaped bidirectional LSTM stack oracle, fp64.  TEST INFRASTRUCTURE ONLY.

PAPER.md §6.3.1 (lines 946-953): DS2 is a stack of (bidirectional) LSTM layers, Echo's recompute
target there being the LSTM feature maps.  Reading R21: the conv front-end is replaced by an
N(0,1) input [T,B,F]; the bidirectional outputs are concatenated to [T,B,2H]; a per-frame
linear layer to 29 classes with mean softmax cross-entropy stands in for CTC.  The reverse
direction runs the oracle LSTM (oracle/lstm.py) over the time-reversed sequence.
Pins: tests/test_oracle_ds2.py (FD; torch.nn.LSTM(bidirectional=True) fp64 autograd).
"""
from __future__ import annotations

import numpy as np

from .lstm import layer_forward, layer_backward


def step(params, batch, cfg, need_grads=True):
    P = {k: np.asarray(v, np.float64) for k, v in params.items()}
    T, B, H = cfg.T, cfg.B, cfg.H
    z = np.zeros((B, H))
    X = np.asarray(batch["x"], np.float64)
    ins = []
    for l in range(cfg.layers):
        ins.append(X)
        hf = layer_forward(X, P[f"l{l}.fw.Wx"], P[f"l{l}.fw.Wh"], P[f"l{l}.fw.b"], z, z)["H"]
        hb = layer_forward(X[::-1], P[f"l{l}.bw.Wx"], P[f"l{l}.bw.Wh"], P[f"l{l}.bw.b"], z, z)["H"][::-1]
        X = np.concatenate([hf, hb], axis=-1)
    logits = X @ P["out.W"].T + P["out.b"]                         # [T, B, classes]
    m = logits.max(axis=-1, keepdims=True)
    logp = logits - m - np.log(np.exp(logits - m).sum(axis=-1, keepdims=True))
    lab = np.asarray(batch["labels"])
    N = T * B
    loss = -np.take_along_axis(logp, lab[..., None], axis=-1).sum() / N
    out = {"loss": float(loss)}
    if not need_grads:
        return out
    G = {}
    dlog = np.exp(logp)
    np.put_along_axis(dlog, lab[..., None], np.take_along_axis(dlog, lab[..., None], axis=-1) - 1.0, axis=-1)
    dlog /= N
    G["out.W"] = dlog.reshape(N, -1).T @ X.reshape(N, -1)
    G["out.b"] = dlog.reshape(N, -1).sum(axis=0)
    dX = dlog @ P["out.W"]
    for l in reversed(range(cfg.layers)):
        Xl = ins[l]
        bf = layer_backward(Xl, P[f"l{l}.fw.Wx"], P[f"l{l}.fw.Wh"], P[f"l{l}.fw.b"], z, z, dX[..., :H])
        bb = layer_backward(Xl[::-1], P[f"l{l}.bw.Wx"], P[f"l{l}.bw.Wh"], P[f"l{l}.bw.b"], z, z, dX[..., H:][::-1])
        for d, r in (("fw", bf), ("bw", bb)):
            G[f"l{l}.{d}.Wx"], G[f"l{l}.{d}.Wh"], G[f"l{l}.{d}.b"] = r["dWx"], r["dWh"], r["db"]
        dX = bf["dX"] + bb["dX"][::-1]
    out["grads"] = G
    return out
