"""Pins for oracle/ds2.py."""
import numpy as np
import torch

from oracle import ds2 as O
from synth.configs import SMALL_DS2
from synth.data import ds2_params, ds2_batch


def test_torch_bidirectional_lstm_crosscheck():
    """torch.nn.LSTM(bidirectional=True) stack + linear + cross-entropy, fp64 autograd."""
    cfg = SMALL_DS2
    P = {k: np.asarray(v, np.float64) for k, v in ds2_params(3, cfg).items()}
    b = ds2_batch(4, cfg)
    r = O.step(P, b, cfg)
    m = torch.nn.LSTM(cfg.F, cfg.H, num_layers=cfg.layers, bidirectional=True).double()
    T = {}
    with torch.no_grad():
        for l in range(cfg.layers):
            for d, suf in (("fw", ""), ("bw", "_reverse")):
                getattr(m, f"weight_ih_l{l}{suf}").copy_(torch.from_numpy(P[f"l{l}.{d}.Wx"]))
                getattr(m, f"weight_hh_l{l}{suf}").copy_(torch.from_numpy(P[f"l{l}.{d}.Wh"]))
                getattr(m, f"bias_ih_l{l}{suf}").copy_(torch.from_numpy(P[f"l{l}.{d}.b"]))
                getattr(m, f"bias_hh_l{l}{suf}").zero_()
    W = torch.from_numpy(P["out.W"]).requires_grad_(True)
    bo = torch.from_numpy(P["out.b"]).requires_grad_(True)
    y, _ = m(torch.from_numpy(np.asarray(b["x"], np.float64)))
    logits = y @ W.T + bo
    loss = torch.nn.functional.cross_entropy(logits.reshape(-1, cfg.classes), torch.from_numpy(b["labels"]).reshape(-1))
    loss.backward()
    assert abs(loss.item() - r["loss"]) < 1e-12
    assert np.abs(W.grad.numpy() - r["grads"]["out.W"]).max() < 1e-12
    for l in range(cfg.layers):
        for d, suf in (("fw", ""), ("bw", "_reverse")):
            g = getattr(m, f"weight_ih_l{l}{suf}").grad.numpy()
            assert np.abs(g - r["grads"][f"l{l}.{d}.Wx"]).max() < 1e-12
            g = getattr(m, f"weight_hh_l{l}{suf}").grad.numpy()
            assert np.abs(g - r["grads"][f"l{l}.{d}.Wh"]).max() < 1e-12


def test_fd_sampled():
    cfg = SMALL_DS2
    P = {k: np.asarray(v, np.float64) for k, v in ds2_params(5, cfg).items()}
    b = ds2_batch(6, cfg)
    G = O.step(P, b, cfg)["grads"]
    g = np.random.default_rng(1)
    eps = 1e-6
    for name, val in P.items():
        for i in g.choice(val.size, size=3, replace=False):
            Pp = {k: v.copy() for k, v in P.items()}
            Pm = {k: v.copy() for k, v in P.items()}
            Pp[name].reshape(-1)[i] += eps
            Pm[name].reshape(-1)[i] -= eps
            num = (O.step(Pp, b, cfg, False)["loss"] - O.step(Pm, b, cfg, False)["loss"]) / (2 * eps)
            assert abs(num - G[name].reshape(-1)[i]) <= 1e-7 + 1e-6 * abs(num), name
