"""Pins for oracle/transformer.py."""
import numpy as np
import torch

from oracle import transformer as O
from synth.configs import SMALL_TX, TXConfig
from synth.data import tx_params, tx_batch


def test_fd_gradients():
    cfg = SMALL_TX
    P = {k: np.asarray(v, np.float64) for k, v in tx_params(1, cfg).items()}
    b = tx_batch(2, cfg)
    keep = O.masks(cfg, b["seeds"])
    G = O.step(P, b, cfg, keep)["grads"]
    g = np.random.default_rng(0)
    eps = 1e-6
    for name, val in P.items():
        for i in g.choice(val.size, size=4, replace=False):
            Pp = {k: v.copy() for k, v in P.items()}
            Pm = {k: v.copy() for k, v in P.items()}
            Pp[name].reshape(-1)[i] += eps
            Pm[name].reshape(-1)[i] -= eps
            num = (O.step(Pp, b, cfg, keep, False)["loss"] - O.step(Pm, b, cfg, keep, False)["loss"]) / (2 * eps)
            assert abs(num - G[name].reshape(-1)[i]) <= 1e-7 + 1e-6 * abs(num), name


def test_single_head_no_dropout_is_plain_attention():
    cfg = TXConfig("t", B=2, L=5, d_model=4, heads=1, blocks=1, dropout_p=0.0)
    P = {k: np.asarray(v, np.float64) for k, v in tx_params(3, cfg).items()}
    b = tx_batch(4, cfg)
    y = O.step(P, b, cfg, need_grads=False)["y"]
    x = torch.from_numpy(np.asarray(b["x"], np.float64))
    T = {k: torch.from_numpy(v) for k, v in P.items()}
    att = torch.softmax((x @ T["b0.Wq"].T) @ (x @ T["b0.Wk"].T).transpose(1, 2) / 2.0, dim=-1)
    ref = (att @ (x @ T["b0.Wv"].T)) @ T["b0.Wo"].T + x
    assert np.abs(y - ref.numpy()).max() < 1e-12
