"""Full NMT training step oracle (loss + every parameter gradient), fp64.
TEST INFRASTRUCTURE ONLY.

Model: PAPER.md §2, lines 125-138 (Fig. 2): embedding -> LSTM encoder whose
hidden states at all steps form H_s [B x T x H] -> decoder that decodes one
target word per step, with attention (1) scores/weights, (2) context, (3)
a_t from [context; query] "sent to the next decoder time step" -> output
layer -> training loss.  Readings: R3 MLP score with qp = W_q h + b_q,
Kp = W_k H_s; R6 zero initial states; R7 a_t = tanh(W_cc ctx_t + W_ch h_t) and
decoder input x_t = [emb(y_{t-1}); a_{t-1}] with a_0 = 0; R10 mean softmax
cross-entropy over all B*Td target tokens; R8 source masking; R31 embedding dropout with rate
cfg.dropout on the source and target embeddings (Philox keep-masks of reading R19, one site per
embedding, keys batch["drop_seeds"], element n = (t*B + b)*E + j of the time-major [T,B,E] tensor);
R33 hidden dropout with rate cfg.dropout_hidden on the inputs of every LSTM layer above the first
(encoder and decoder: the layer below's h) and on a_t where it enters the output layer (not on the
input-feeding path), keys batch["drop_seeds"][2:] in the order encoder l = 0..Le-2, decoder l =
0..Ld-2, output; element n = (t*B + b)*H + j of the time-major [T,B,H] tensor.

Echo changes no math, so this is the one oracle for both the
STASH and RECOMPUTE GPU modes.  Pins: tests/test_oracle_nmt.py (central finite
differences of the loss, torch fp64 autograd of the same forward).
"""
from __future__ import annotations

import numpy as np

from . import attention
from .dot_softmax import dropout_keep_mask
from .lstm import cell_forward, cell_backward, layer_forward, layer_backward


def _f64(params):
    return {k: np.asarray(v, np.float64) for k, v in params.items()}


def _logsoftmax(z):
    m = z.max(axis=1, keepdims=True)
    return z - m - np.log(np.exp(z - m).sum(axis=1, keepdims=True))


def hidden_masks(cfg, batch):
    """R33 keep-masks scaled by 1 / (1 - p) (all ones when cfg.dropout_hidden == 0): encoder [Le-1] x
    [Ts,B,H], decoder [Ld-1] x [Td,B,H], output [Td,B,H]."""
    B, Ts, Td, H = cfg.B, cfg.Ts, cfg.Td, cfg.H
    q = getattr(cfg, "dropout_hidden", 0.0)
    Le, Ld = cfg.enc_layers, cfg.dec_layers
    if q <= 0.0:
        return [np.ones((Ts, B, H))] * (Le - 1), [np.ones((Td, B, H))] * (Ld - 1), np.ones((Td, B, H))
    keys = [int(x) for x in batch["drop_seeds"][2:]]
    mk = lambda key, T: dropout_keep_mask(key, 0, T * B * H, q).reshape(T, B, H) / (1.0 - q)
    me = [mk(keys[l], Ts) for l in range(Le - 1)]
    md = [mk(keys[Le - 1 + l], Td) for l in range(Ld - 1)]
    return me, md, mk(keys[Le - 1 + Ld - 1], Td)


def step(params, batch, cfg, need_grads=True):
    """Returns {"loss": float, "grads": {name: array}, "trace": intermediates}."""
    P = _f64(params)
    src, tgt_in, tgt_out, src_len = batch["src"], batch["tgt_in"], batch["tgt_out"], batch["src_len"]
    B, Ts, Td, E, H = cfg.B, cfg.Ts, cfg.Td, cfg.E, cfg.H
    zeros = np.zeros((B, H))
    p = getattr(cfg, "dropout", 0.0)
    if p > 0.0:                                              # R31: keep / (1 - p) per embedding element
        ks, kt = (int(x) for x in batch["drop_seeds"][:2])
        ms = dropout_keep_mask(ks, 0, Ts * B * E, p).reshape(Ts, B, E) / (1.0 - p)
        mt = dropout_keep_mask(kt, 0, Td * B * E, p).reshape(Td, B, E) / (1.0 - p)
    else:
        ms, mt = np.ones((Ts, B, E)), np.ones((Td, B, E))
    me, md, mo = hidden_masks(cfg, batch)

    # ---------------- encoder
    X = P["emb_src"][src].transpose(1, 0, 2) * ms            # [Ts, B, E]
    enc_in = []
    for l in range(cfg.enc_layers):
        if l > 0:
            X = X * me[l - 1]                                # R33: dropout on the layer below's h
        enc_in.append(X)
        fw = layer_forward(X, P[f"enc{l}.Wx"], P[f"enc{l}.Wh"], P[f"enc{l}.b"], zeros, zeros)
        X = fw["H"]
    Hs = X.transpose(1, 0, 2)                                # [B, Ts, H] source hidden state
    Kp = Hs @ P["att.Wk"].T                                  # [B, Ts, A]

    # ---------------- decoder with attention and input feeding
    L = cfg.dec_layers
    h = [zeros.copy() for _ in range(L)]
    c = [zeros.copy() for _ in range(L)]
    a_prev = zeros.copy()
    tr = {"A": [[None] * Td for _ in range(L)], "c_prev": [[None] * Td for _ in range(L)],
          "h_prev": [[None] * Td for _ in range(L)], "x_in": [[None] * Td for _ in range(L)],
          "q": [None] * Td, "qp": [None] * Td, "ctx": [None] * Td, "a": [None] * Td, "logp": [None] * Td}
    loss = 0.0
    for t in range(Td):
        x = np.concatenate([P["emb_tgt"][tgt_in[:, t]] * mt[t], a_prev], axis=1)
        for l in range(L):
            A = x @ P[f"dec{l}.Wx"].T + h[l] @ P[f"dec{l}.Wh"].T + P[f"dec{l}.b"]
            tr["A"][l][t], tr["c_prev"][l][t], tr["h_prev"][l][t], tr["x_in"][l][t] = A, c[l], h[l], x
            s = cell_forward(A, c[l])
            h[l], c[l] = s["h"], s["c"]
            x = s["h"] * md[l][t] if l < L - 1 else s["h"]   # R33: input of the layer above
        q = x                                                # the query
        qp = q @ P["att.Wq"].T + P["att.bq"]
        ctx = attention.forward(qp, Kp, P["att.v"], Hs, src_len)["ctx"]
        a = np.tanh(ctx @ P["att.Wcc"].T + q @ P["att.Wch"].T)   # (3) attention hidden state a_t
        logits = (a * mo[t]) @ P["out.Wo"].T + P["out.bo"]     # R33: dropout where a_t enters the output layer
        logp = _logsoftmax(logits)
        loss -= logp[np.arange(B), tgt_out[:, t]].sum()
        tr["q"][t], tr["qp"][t], tr["ctx"][t], tr["a"][t], tr["logp"][t] = q, qp, ctx, a, logp
        a_prev = a
    N = B * Td
    loss /= N
    out = {"loss": loss, "trace": tr, "Hs": Hs, "Kp": Kp}
    if not need_grads:
        return out

    # ---------------- backward (BPTT; FC grads per Eq. 2)
    G = {k: np.zeros_like(v) for k, v in P.items()}
    dh_rec = [zeros.copy() for _ in range(L)]
    dc = [zeros.copy() for _ in range(L)]
    da_carry = zeros.copy()
    dKp = np.zeros_like(Kp)
    dHs = np.zeros_like(Hs)
    for t in reversed(range(Td)):
        dlogits = np.exp(tr["logp"][t])
        dlogits[np.arange(B), tgt_out[:, t]] -= 1.0
        dlogits /= N
        a, q, ctx = tr["a"][t], tr["q"][t], tr["ctx"][t]
        G["out.Wo"] += dlogits.T @ (a * mo[t])
        G["out.bo"] += dlogits.sum(axis=0)
        da = (dlogits @ P["out.Wo"]) * mo[t] + da_carry
        dpre = da * (1.0 - a * a)
        G["att.Wcc"] += dpre.T @ ctx
        G["att.Wch"] += dpre.T @ q
        dctx = dpre @ P["att.Wcc"]
        dq = dpre @ P["att.Wch"]
        ab = attention.backward(tr["qp"][t], Kp, P["att.v"], Hs, dctx, src_len)
        dKp += ab["dKp"]
        dHs += ab["dHs"]
        G["att.v"] += ab["dv"]
        G["att.Wq"] += ab["dqp"].T @ q
        G["att.bq"] += ab["dqp"].sum(axis=0)
        dx = dq + ab["dqp"] @ P["att.Wq"]
        for l in reversed(range(L)):
            dh = dx + dh_rec[l]
            dA, dc[l] = cell_backward(tr["A"][l][t], tr["c_prev"][l][t], dh, dc[l])
            G[f"dec{l}.Wh"] += dA.T @ tr["h_prev"][l][t]
            G[f"dec{l}.Wx"] += dA.T @ tr["x_in"][l][t]
            G[f"dec{l}.b"] += dA.sum(axis=0)
            dh_rec[l] = dA @ P[f"dec{l}.Wh"]
            dx = dA @ P[f"dec{l}.Wx"]
            if l > 0:
                dx = dx * md[l - 1][t]                       # through the R33 dropout below
        np.add.at(G["emb_tgt"], tgt_in[:, t], dx[:, :E] * mt[t])
        da_carry = dx[:, E:]
    G["att.Wk"] += np.einsum("bsa,bsh->ah", dKp, Hs)
    dHs += dKp @ P["att.Wk"]
    dH = dHs.transpose(1, 0, 2)                              # [Ts, B, H]
    for l in reversed(range(cfg.enc_layers)):
        bw = layer_backward(enc_in[l], P[f"enc{l}.Wx"], P[f"enc{l}.Wh"], P[f"enc{l}.b"], zeros, zeros, dH)
        G[f"enc{l}.Wx"] += bw["dWx"]
        G[f"enc{l}.Wh"] += bw["dWh"]
        G[f"enc{l}.b"] += bw["db"]
        dH = bw["dX"] * me[l - 1] if l > 0 else bw["dX"]
    np.add.at(G["emb_src"], src.T.reshape(-1), (dH * ms).reshape(Ts * B, E))
    out["grads"] = G
    return out
