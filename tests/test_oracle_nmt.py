"""Pins for oracle/nmt.py: full training-step loss and gradients."""
import numpy as np
import torch

from oracle import nmt as O
from synth.configs import NMTConfig, C1, SMALL_NMT
from synth.data import nmt_params, nmt_batch


def _f64(p):
    return {k: np.asarray(v, np.float64) for k, v in p.items()}


def test_zero_weights_closed_form():
    """All weights/biases 0 => h = a = 0, logits = 0 => loss = ln V; dbo = mean(softmax - onehot)."""
    cfg = C1
    P = {k: np.zeros_like(v, dtype=np.float64) for k, v in nmt_params(0, cfg).items()}
    b = nmt_batch(1, cfg, lengths="random")
    r = O.step(P, b, cfg)
    assert abs(r["loss"] - np.log(cfg.V)) < 1e-14
    counts = np.bincount(b["tgt_out"].reshape(-1), minlength=cfg.V)
    expect = (1.0 / cfg.V) - counts / (cfg.B * cfg.Td)
    assert np.abs(r["grads"]["out.bo"] - expect).max() < 1e-15
    assert np.all(r["grads"]["out.Wo"] == 0)


def test_fd_sampled_gradients_c1():
    cfg = C1
    P = _f64(nmt_params(3, cfg))
    b = nmt_batch(4, cfg, lengths="random")
    G = O.step(P, b, cfg)["grads"]
    g = np.random.default_rng(0)
    eps = 1e-6
    for name, val in P.items():
        flat = val.reshape(-1)
        idxs = g.choice(flat.size, size=min(4, flat.size), replace=False)
        if name.startswith("emb"):   # pick rows that are actually used
            toks = b["src"] if name == "emb_src" else b["tgt_in"]
            row = int(toks.reshape(-1)[0])
            idxs = np.array([row * val.shape[1] + j for j in range(3)])
        for i in idxs:
            Pp = {k: v.copy() for k, v in P.items()}
            Pm = {k: v.copy() for k, v in P.items()}
            Pp[name].reshape(-1)[i] += eps
            Pm[name].reshape(-1)[i] -= eps
            num = (O.step(Pp, b, cfg, False)["loss"] - O.step(Pm, b, cfg, False)["loss"]) / (2 * eps)
            ana = G[name].reshape(-1)[i]
            assert abs(num - ana) <= 1e-7 + 1e-6 * abs(num), (name, i, num, ana)


def _torch_nmt_loss(P, b, cfg, ms=None, mt=None, hm=None):
    """Same model written with torch.nn.LSTM / LSTMCell + autograd (library routines).  ms / mt:
    optional embedding-dropout multipliers [Ts,B,E] / [Td,B,E] (keep / (1 - p)); hm: optional R33
    multipliers (encoder list, decoder list, output), applied where the layer above / the output
    layer reads h / a_t."""
    T = {k: torch.from_numpy(v).requires_grad_(True) for k, v in P.items()}
    B, H, E = cfg.B, cfg.H, cfg.E
    x = T["emb_src"][torch.from_numpy(b["src"])].transpose(0, 1)
    if ms is not None:
        x = x * torch.from_numpy(ms)
    for l in range(cfg.enc_layers):
        if hm is not None and l > 0:
            x = x * torch.from_numpy(hm[0][l - 1])
        m = torch.nn.LSTM(x.shape[2], H).double()
        x, _ = torch.func.functional_call(m, {"weight_ih_l0": T[f"enc{l}.Wx"], "weight_hh_l0": T[f"enc{l}.Wh"],
                                              "bias_ih_l0": T[f"enc{l}.b"], "bias_hh_l0": torch.zeros(4 * H, dtype=torch.float64)}, (x,))
    Hs = x.transpose(0, 1)
    Kp = Hs @ T["att.Wk"].T
    valid = torch.arange(cfg.Ts)[None, :] < torch.from_numpy(b["src_len"]).long()[:, None]
    cells = [torch.nn.LSTMCell(E + H if l == 0 else H, H).double() for l in range(cfg.dec_layers)]
    h = [torch.zeros(B, H, dtype=torch.float64) for _ in cells]
    c = [torch.zeros(B, H, dtype=torch.float64) for _ in cells]
    a = torch.zeros(B, H, dtype=torch.float64)
    loss = 0
    for t in range(cfg.Td):
        et = T["emb_tgt"][torch.from_numpy(b["tgt_in"][:, t])]
        if mt is not None:
            et = et * torch.from_numpy(mt[t])
        inp = torch.cat([et, a], dim=1)
        for l, cell in enumerate(cells):
            h[l], c[l] = torch.func.functional_call(cell, {"weight_ih": T[f"dec{l}.Wx"], "weight_hh": T[f"dec{l}.Wh"],
                                                          "bias_ih": T[f"dec{l}.b"], "bias_hh": torch.zeros(4 * H, dtype=torch.float64)},
                                                    (inp, (h[l], c[l])))
            inp = h[l] * torch.from_numpy(hm[1][l][t]) if hm is not None and l < cfg.dec_layers - 1 else h[l]
        q = inp
        qp = q @ T["att.Wq"].T + T["att.bq"]
        sc = torch.tanh(qp[:, None, :] + Kp) @ T["att.v"]
        alpha = torch.softmax(sc.masked_fill(~valid, float("-inf")), dim=1)
        ctx = torch.einsum("bs,bsk->bk", alpha, Hs)
        a = torch.tanh(ctx @ T["att.Wcc"].T + q @ T["att.Wch"].T)
        logits = (a * torch.from_numpy(hm[2][t]) if hm is not None else a) @ T["out.Wo"].T + T["out.bo"]
        loss = loss + torch.nn.functional.cross_entropy(logits, torch.from_numpy(b["tgt_out"][:, t]), reduction="sum")
    loss = loss / (B * cfg.Td)
    loss.backward()
    return loss.item(), {k: v.grad.numpy() for k, v in T.items()}


def test_torch_autograd_crosscheck_small_nmt():
    cfg = SMALL_NMT
    P = _f64(nmt_params(5, cfg))
    b = nmt_batch(6, cfg, lengths="random")
    r = O.step(P, b, cfg)
    tl, tg = _torch_nmt_loss(P, b, cfg)
    assert abs(r["loss"] - tl) < 1e-12
    for k in P:
        scale = max(np.abs(tg[k]).max(), 1e-30)
        assert np.abs(r["grads"][k] - tg[k]).max() / scale < 1e-10, k


def test_embedding_dropout_oracle_pins():
    """R31 embedding dropout: (1) the same model in torch autograd with the masks applied explicitly
    (the mask generator itself is pinned by the Random123 known-answer vectors in
    test_oracle_dot_softmax.py); (2) central FD on C1 with p = 0.3; (3) p = 0 equals no dropout."""
    from dataclasses import replace
    from oracle.dot_softmax import dropout_keep_mask
    cfg = replace(SMALL_NMT, dropout=0.25)
    P = _f64(nmt_params(5, cfg))
    b = nmt_batch(6, cfg, lengths="random")
    r = O.step(P, b, cfg)
    ks, kt = (int(x) for x in b["drop_seeds"])
    ms = dropout_keep_mask(ks, 0, cfg.Ts * cfg.B * cfg.E, 0.25).reshape(cfg.Ts, cfg.B, cfg.E) / 0.75
    mt = dropout_keep_mask(kt, 0, cfg.Td * cfg.B * cfg.E, 0.25).reshape(cfg.Td, cfg.B, cfg.E) / 0.75
    assert 0.6 < (ms > 0).mean() < 0.9 and 0.6 < (mt > 0).mean() < 0.9
    tl, tg = _torch_nmt_loss(P, b, cfg, ms, mt)
    assert abs(r["loss"] - tl) < 1e-12
    for k in P:
        scale = max(np.abs(tg[k]).max(), 1e-30)
        assert np.abs(r["grads"][k] - tg[k]).max() / scale < 1e-10, k
    c1 = replace(C1, dropout=0.3)
    P1 = _f64(nmt_params(3, c1))
    b1 = nmt_batch(4, c1)
    G = O.step(P1, b1, c1)["grads"]
    eps = 1e-6
    for name in ("emb_src", "emb_tgt", "enc0.Wx", "dec0.Wx"):
        toks = b1["src"] if name == "emb_src" else b1["tgt_in"]
        idxs = [int(toks.reshape(-1)[0]) * P1[name].shape[1] + j for j in range(4)] if name.startswith("emb") else [0, 7, 33]
        for i in idxs:
            Pp = {k: v.copy() for k, v in P1.items()}
            Pm = {k: v.copy() for k, v in P1.items()}
            Pp[name].reshape(-1)[i] += eps
            Pm[name].reshape(-1)[i] -= eps
            num = (O.step(Pp, b1, c1, False)["loss"] - O.step(Pm, b1, c1, False)["loss"]) / (2 * eps)
            assert abs(num - G[name].reshape(-1)[i]) <= 1e-7 + 1e-6 * abs(num), (name, i)
    r0 = O.step(P1, b1, replace(c1, dropout=0.0))
    r00 = O.step(P1, b1, C1)
    assert r0["loss"] == r00["loss"]


def test_hidden_dropout_oracle_pins():
    """R33 hidden dropout (inter-layer LSTM inputs, a_t into the output layer): (1) torch autograd of
    the same model with the masks applied explicitly at those points, every gradient to 1e-10; (2) the
    masks keep ~(1 - p) of the elements and are distinct per site; (3) central FD on a 2+2-layer tiny
    config; (4) p = 0 equals no dropout."""
    from dataclasses import replace
    cfg = replace(SMALL_NMT, dropout=0.2, dropout_hidden=0.3)
    P = _f64(nmt_params(5, cfg))
    b = nmt_batch(6, cfg, lengths="random")
    assert len(b["drop_seeds"]) == 2 + cfg.hidden_drop_sites() == 5
    r = O.step(P, b, cfg)
    from oracle.dot_softmax import dropout_keep_mask
    ks, kt = (int(x) for x in b["drop_seeds"][:2])
    ms = dropout_keep_mask(ks, 0, cfg.Ts * cfg.B * cfg.E, 0.2).reshape(cfg.Ts, cfg.B, cfg.E) / 0.8
    mt = dropout_keep_mask(kt, 0, cfg.Td * cfg.B * cfg.E, 0.2).reshape(cfg.Td, cfg.B, cfg.E) / 0.8
    hm = O.hidden_masks(cfg, b)
    for m in hm[0] + hm[1] + [hm[2]]:
        assert 0.55 < (m > 0).mean() < 0.85
    assert not np.array_equal(hm[1][0] > 0, hm[2] > 0)
    tl, tg = _torch_nmt_loss(P, b, cfg, ms, mt, hm)
    assert abs(r["loss"] - tl) < 1e-12
    for k in P:
        scale = max(np.abs(tg[k]).max(), 1e-30)
        assert np.abs(r["grads"][k] - tg[k]).max() / scale < 1e-10, k
    tiny = NMTConfig("tiny2", B=2, Ts=3, Td=3, E=8, H=8, A=8, V=11, enc_layers=2, dec_layers=2, dropout_hidden=0.4)
    P1 = _f64(nmt_params(3, tiny))
    b1 = nmt_batch(4, tiny)
    G = O.step(P1, b1, tiny)["grads"]
    eps = 1e-6
    for name in ("enc0.Wx", "enc1.Wx", "dec0.Wh", "dec1.Wx", "out.Wo", "att.Wq"):
        for i in (0, 5, 17):
            Pp = {k: v.copy() for k, v in P1.items()}
            Pm = {k: v.copy() for k, v in P1.items()}
            Pp[name].reshape(-1)[i] += eps
            Pm[name].reshape(-1)[i] -= eps
            num = (O.step(Pp, b1, tiny, False)["loss"] - O.step(Pm, b1, tiny, False)["loss"]) / (2 * eps)
            assert abs(num - G[name].reshape(-1)[i]) <= 1e-7 + 1e-6 * abs(num), (name, i)
    assert O.step(P1, b1, replace(tiny, dropout_hidden=0.0))["loss"] == \
        O.step(P1, {k: v for k, v in b1.items() if k != "drop_seeds"} | {"drop_seeds": b1["drop_seeds"][:2]},
               replace(tiny, dropout_hidden=0.0))["loss"]
