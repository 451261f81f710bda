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


def test_multi_head_dropout_matches_torch_per_head_slices():
    """Multi-head split / merge pin: heads = 4, p = 0.1, two blocks.  The torch
    model below defines head h as the COLUMN SLICE [h*dh, (h+1)*dh) of Q, K, V (no reshape), runs
    torch.softmax per head, applies the same explicit keep-mask m[k][:, h] with scale 1/(1-p), and
    concatenates the per-head outputs along columns before W_o (R27).  Forward y and
    every gradient (torch autograd, fp64) must match the oracle.  A reshape that mixes positions
    across heads, a transposed head layout or a mask indexed by the wrong head fails here."""
    cfg = TXConfig("mh", B=2, L=6, d_model=16, heads=4, blocks=2, dropout_p=0.1)
    P = {k: np.asarray(v, np.float64) for k, v in tx_params(5, cfg).items()}
    b = tx_batch(6, cfg)
    keep = O.masks(cfg, b["seeds"])
    assert 0 < sum(int((~m.astype(bool)).sum()) for m in keep)          # some entries are dropped
    ref = O.step(P, b, cfg, keep)

    T = {k: torch.from_numpy(v.copy()).requires_grad_(True) for k, v in P.items()}
    x = torch.from_numpy(np.asarray(b["x"], np.float64))
    dh = cfg.d_model // cfg.heads
    for k in range(cfg.blocks):
        Q, K, V = x @ T[f"b{k}.Wq"].T, x @ T[f"b{k}.Wk"].T, x @ T[f"b{k}.Wv"].T
        outs = []
        for h in range(cfg.heads):
            cols = slice(h * dh, (h + 1) * dh)
            att = torch.softmax(Q[:, :, cols] @ K[:, :, cols].transpose(1, 2) / np.sqrt(dh), dim=-1)
            m = torch.from_numpy(np.asarray(keep[k][:, h], np.float64))
            outs.append((att * m / (1.0 - cfg.dropout_p)) @ V[:, :, cols])
        x = torch.cat(outs, dim=-1) @ T[f"b{k}.Wo"].T + x
    loss = (x @ T["out.r"]).sum() / (cfg.B * cfg.L)
    loss.backward()
    assert abs(loss.item() - ref["loss"]) < 1e-12
    assert np.abs(x.detach().numpy() - ref["y"]).max() < 1e-12
    for name, t in T.items():
        g = t.grad.numpy()
        assert np.abs(g - ref["grads"][name]).max() <= 1e-12 * max(1.0, np.abs(g).max()), name
