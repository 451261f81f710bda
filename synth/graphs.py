"""Graph documents for the footprint estimator (structure and shapes only; no estimator logic).

Schema:
  {"version": 1,
   "placeholders": [{"id", "name", "shape", "dtype", "trainable", "tag"}],
   "nodes": [{"id", "op", "inputs": [[node, out], ...], "attrs": {...}, "tag"}],
   "outputs": [[node, out], ...]}
Ids are dense over placeholders and nodes together, and every node's inputs reference
earlier ids (so id order is a topological order).  dtypes: f32, bf16, f64, i32, i64, bit.

Builders: the paper's worked examples (Fig. 6/9 add_tanh, Fig. 7/10 broadcast_attn,
Fig. 12 tanh->FC, Fig. 4 chain), an unfused LSTM layer, one MLP-attention step, the NMT
model with the op structure of the GPU path (paper_1805_08899_b200/nmt.py), and seeded
random graphs.
"""
from __future__ import annotations

import json

import numpy as np


class GraphBuilder:
    def __init__(self):
        self.placeholders = []
        self.nodes = []
        self.outputs = []
        self.n = 0

    def placeholder(self, name, shape, dtype="f32", trainable=False, tag=""):
        i = self.n
        self.n += 1
        self.placeholders.append({"id": i, "name": name, "shape": list(map(int, shape)), "dtype": dtype,
                                  "trainable": bool(trainable), "tag": tag})
        return (i, 0)

    def op(self, op, inputs, tag="", nout=1, **attrs):
        i = self.n
        self.n += 1
        self.nodes.append({"id": i, "op": op, "inputs": [list(e) for e in inputs], "attrs": attrs, "tag": tag})
        if nout == 1:
            return (i, 0)
        return tuple((i, k) for k in range(nout))

    def output(self, e):
        self.outputs.append(list(e))

    def doc(self):
        return {"version": 1, "placeholders": self.placeholders, "nodes": self.nodes, "outputs": self.outputs}

    def json(self):
        return json.dumps(self.doc())


# ----------------------------------------------------------------------------- paper worked examples
def add_tanh(N=1024, dtype="f32"):
    """Fig. 6: Z = tanh(X + Y), loss = sum(Z)."""
    g = GraphBuilder()
    X = g.placeholder("X", [N], dtype)
    Y = g.placeholder("Y", [N], dtype)
    Z = g.op("tanh", [g.op("add", [X, Y])])
    g.output(g.op("sum_reduce", [Z]))
    return g.doc()


def broadcast_attn(T=64, N=256, dtype="f32"):
    """Fig. 7/10: T tensors [N] broadcast-added with one shared [T x N], then tanh."""
    g = GraphBuilder()
    K = g.placeholder("K", [T, N], dtype)
    qs = [g.placeholder(f"q{t}", [N], dtype) for t in range(T)]
    loss = None
    for t in range(T):
        y = g.op("tanh", [g.op("broadcast_add", [qs[t], K])])
        s = g.op("sum_reduce", [y])
        loss = s if loss is None else g.op("add", [loss, s])
    g.output(loss)
    return g.doc()


def tanh_fc(B=8, H=16, dtype="f32"):
    """Fig. 12: a cheap producer (broadcast-add with a weight, then tanh) feeding an FC whose
    gradient needs only its input (Eq. 2)."""
    g = GraphBuilder()
    q = g.placeholder("q", [H], dtype)
    K = g.placeholder("K", [B, H], dtype, trainable=True)
    W = g.placeholder("W", [H, H], dtype, trainable=True)
    t = g.op("tanh", [g.op("broadcast_add", [q, K])])
    y = g.op("fully_connected", [t, W])
    g.output(g.op("sum_reduce", [y]))
    return g.doc()


def chain4(N=64, dtype="f32"):
    """Fig. 4: a chain of four cheap nodes whose gradients need their outputs."""
    g = GraphBuilder()
    x = g.placeholder("x", [N], dtype)
    e = x
    for _ in range(4):
        e = g.op("tanh", [e])
    g.output(g.op("sum_reduce", [e]))
    return g.doc()


# ----------------------------------------------------------------------------- LSTM / attention pieces
def lstm_cell(g, x_gx, h_prev, c_prev, Wh, H, B, s="f32", tag="rnn", gh=True, extra=None):
    """Non-linear block f of one cell with the GPU path's op structure:
    A = gx (+ gh) ; 4 slices ; sigma/tanh ; c = f*c_prev + i*g (fp32) ; h = o * tanh(c)."""
    A = x_gx
    if extra is not None:
        A = g.op("add", [A, extra], tag=tag)
    if gh:
        A = g.op("add", [A, g.op("fully_connected", [h_prev, Wh], tag=tag)], tag=tag)
    i_p, f_p, g_p, o_p = (g.op("slice", [A], tag=tag, axis=1, begin=k * H, end=(k + 1) * H) for k in range(4))
    i = g.op("sigmoid", [i_p], tag=tag)
    f = g.op("sigmoid", [f_p], tag=tag)
    gg = g.op("tanh", [g_p], tag=tag)
    o = g.op("sigmoid", [o_p], tag=tag)
    fc = g.op("mul", [f, c_prev], tag=tag, dtype="f32")
    ig = g.op("mul", [i, gg], tag=tag, dtype="f32")
    c = g.op("add", [fc, ig], tag=tag, dtype="f32")
    tc = g.op("tanh", [c], tag=tag, dtype=s)
    h = g.op("mul", [o, tc], tag=tag, dtype=s)
    return h, c


def lstm_layer(T=3, B=2, H=8, I=8, s="f32"):
    """One unrolled LSTM layer with a linear loss on every h_t (T3 in DESIGN.md)."""
    g = GraphBuilder()
    Wx = g.placeholder("Wx", [4 * H, I], s, trainable=True)
    Wh = g.placeholder("Wh", [4 * H, H], s, trainable=True)
    b = g.placeholder("b", [4 * H], "f32", trainable=True)
    h = g.placeholder("h0", [B, H], s)
    c = g.placeholder("c0", [B, H], "f32")
    loss = None
    for t in range(T):
        x = g.placeholder(f"x{t}", [B, I], s)
        gx = g.op("fully_connected", [x, Wx, b], tag="rnn")
        h, c = lstm_cell(g, gx, h, c, Wh, H, B, s)
        Wo = g.placeholder(f"Wo{t}", [1, H], s, trainable=True)
        l = g.op("sum_reduce", [g.op("fully_connected", [h, Wo])])
        loss = l if loss is None else g.op("add", [loss, l])
    g.output(loss)
    return g.doc()


def nmt(cfg, s="f32"):
    """NMT training graph with the op structure of the GPU path (paper_1805_08899_b200/nmt.py).

    Encoder: per step x_t = embedding(slice(src, t)); per layer FC(x) [+ FC(h)] -> cell.
    H_s = stack(h^top_1..h^top_Ts) (a view: the encoder writes h_t into it); Kp = FC(H_s, Wk, bq).
    Decoder step t: e_t = embedding(slice(tgt_in, t)); layer 0: FC(e_t, W_e, b) [+ FC(a_{t-1}, W_a)]
    [+ FC(h_{t-1}, Wh)]; layers > 0: FC(h^{l-1}_t, Wx, b) [+ FC(h_{t-1}, Wh)]; qp = FC(q, Wq);
    z = broadcast_add(qp, Kp); E = tanh(z); sc = dot_last(E, v); alpha = masked_softmax(sc, len);
    ctx = weighted_sum(alpha, H_s); a_t = tanh(FC(ctx, Wcc) + FC(q, Wch)).
    Output: A = stack(a_1..a_Td); logits = FC(A, Wo, bo); softmax_ce_loss(logits, labels) -> loss.
    """
    B, Ts, Td, E, H, A, V = cfg.B, cfg.Ts, cfg.Td, cfg.E, cfg.H, cfg.A, cfg.V
    g = GraphBuilder()
    src = g.placeholder("src", [Ts, B], "i64")
    tgt = g.placeholder("tgt_in", [Td, B], "i64")
    labels = g.placeholder("tgt_out", [Td * B], "i64")
    slen = g.placeholder("src_len", [B], "i32")
    h0 = g.placeholder("h0", [B, H], s)
    c0 = g.placeholder("c0", [B, H], "f32")
    emb_s = g.placeholder("emb_src", [V, E], s, trainable=True)
    emb_t = g.placeholder("emb_tgt", [V, E], s, trainable=True)
    enc = []
    for l in range(cfg.enc_layers):
        I = E if l == 0 else H
        enc.append(tuple(g.placeholder(f"enc{l}.{n}", shp, dt, trainable=True) for n, shp, dt in
                         (("Wx", [4 * H, I], s), ("Wh", [4 * H, H], s), ("b", [4 * H], "f32"))))
    dec = []
    for l in range(cfg.dec_layers):
        if l == 0:
            dec.append(tuple(g.placeholder(f"dec0.{n}", shp, dt, trainable=True) for n, shp, dt in
                             (("We", [4 * H, E], s), ("Wa", [4 * H, H], s), ("Wh", [4 * H, H], s), ("b", [4 * H], "f32"))))
        else:
            dec.append(tuple(g.placeholder(f"dec{l}.{n}", shp, dt, trainable=True) for n, shp, dt in
                             (("Wx", [4 * H, H], s), ("Wh", [4 * H, H], s), ("b", [4 * H], "f32"))))
    Wq = g.placeholder("att.Wq", [A, H], s, trainable=True)
    Wk = g.placeholder("att.Wk", [A, H], s, trainable=True)
    bq = g.placeholder("att.bq", [A], "f32", trainable=True)
    v = g.placeholder("att.v", [A], s, trainable=True)
    Wcc = g.placeholder("att.Wcc", [H, H], s, trainable=True)
    Wch = g.placeholder("att.Wch", [H, H], s, trainable=True)
    Wo = g.placeholder("out.Wo", [V, H], s, trainable=True)
    bo = g.placeholder("out.bo", [V], "f32", trainable=True)
    p = getattr(cfg, "dropout", 0.0)

    def drop(x):                                         # R31: embedding dropout (keep-mask = output 1)
        return g.op("dropout", [x], tag="embed", nout=2, p=p)[0] if p > 0 else x

    ph = getattr(cfg, "dropout_hidden", 0.0)

    def hdrop(x, tag):                                   # R33: inter-layer / output dropout
        return g.op("dropout", [x], tag=tag, nout=2, p=ph)[0] if ph > 0 else x

    # encoder
    xs = [drop(g.op("embedding", [g.op("slice", [src], tag="embed", axis=0, begin=t, end=t + 1, squeeze=1), emb_s],
                    tag="embed")) for t in range(Ts)]
    for l in range(cfg.enc_layers):
        Wx, Wh, b = enc[l]
        h, c = h0, c0
        hs = []
        for t in range(Ts):
            gx = g.op("fully_connected", [xs[t], Wx, b], tag="rnn")
            h, c = lstm_cell(g, gx, h, c, Wh, H, B, s, tag="rnn")
            hs.append(h)
        xs = [hdrop(h, "rnn") for h in hs] if l < cfg.enc_layers - 1 else hs
    Hs = g.op("stack", xs, tag="rnn")                                          # [Ts, B, H]
    Kp = g.op("fully_connected", [Hs, Wk, bq], tag="attention")               # [Ts, B, A]
    # decoder
    hst = [h0] * cfg.dec_layers
    cst = [c0] * cfg.dec_layers
    a_prev = None
    a_all = []
    for t in range(Td):
        e_t = drop(g.op("embedding", [g.op("slice", [tgt], tag="embed", axis=0, begin=t, end=t + 1, squeeze=1), emb_t],
                        tag="embed"))
        x = None
        for l in range(cfg.dec_layers):
            if l == 0:
                We, Wa, Wh, b = dec[0]
                gx = g.op("fully_connected", [e_t, We, b], tag="rnn")
                extra = g.op("fully_connected", [a_prev, Wa], tag="rnn") if a_prev is not None else None
            else:
                Wx, Wh, b = dec[l]
                gx = g.op("fully_connected", [x, Wx, b], tag="rnn")
                extra = None
            h, c = lstm_cell(g, gx, hst[l], cst[l], Wh, H, B, s, tag="rnn", gh=(t > 0), extra=extra)
            hst[l], cst[l] = h, c
            x = hdrop(h, "rnn") if l < cfg.dec_layers - 1 else h
        q = x
        qp = g.op("fully_connected", [q, Wq], tag="attention")                 # [B, A]
        z = g.op("broadcast_add", [qp, Kp], tag="attention")                  # [Ts, B, A]
        Et = g.op("tanh", [z], tag="attention")
        sc = g.op("dot_last", [Et, v], tag="attention")                        # [Ts, B]
        al = g.op("masked_softmax", [sc, slen], tag="attention", dtype="f32")  # [Ts, B]
        ctx = g.op("weighted_sum", [al, Hs], tag="attention", dtype=s)         # [B, H]
        pre = g.op("add", [g.op("fully_connected", [ctx, Wcc], tag="attention"),
                           g.op("fully_connected", [q, Wch], tag="attention")], tag="attention")
        a_t = g.op("tanh", [pre], tag="attention")
        a_all.append(a_t)
        a_prev = a_t
    Aall = g.op("stack", a_all, tag="output")                                  # [Td, B, H]
    logits = g.op("fully_connected", [hdrop(Aall, "output"), Wo, bo], tag="output", dtype="f32")   # [Td, B, V]
    loss, probs = g.op("softmax_ce_loss", [logits, labels], tag="output", nout=2)
    g.output(loss)
    return g.doc()


def ds2(cfg, s="f32"):
    """DeepSpeech2-shaped bidirectional LSTM stack with the op structure of the GPU path
    (paper_1805_08899_b200/ds2.py): per step and direction gx = FC(x_t) or FC(hf_t, Wa) + FC(hb_t, Wb),
    plus FC(h_{t-1}, Wh) (h0 at the first step); per-frame logits = FC(hf_t, Wo_a, b) + FC(hb_t, Wo_b),
    stacked, softmax cross-entropy."""
    T, B, F, H, C = cfg.T, cfg.B, cfg.F, cfg.H, cfg.classes
    g = GraphBuilder()
    x = g.placeholder("x", [T, B, F], s)
    labels = g.placeholder("labels", [T * B], "i64")
    h0 = g.placeholder("h0", [B, H], s)
    c0 = g.placeholder("c0", [B, H], "f32")
    xs = [g.op("slice", [x], tag="input", axis=0, begin=t, end=t + 1, squeeze=1) for t in range(T)]
    low = None
    for l in range(cfg.layers):
        outs = {}
        for d in ("fw", "bw"):
            if l == 0:
                Wx = g.placeholder(f"l{l}.{d}.Wx", [4 * H, F], s, trainable=True)
            else:
                Wa = g.placeholder(f"l{l}.{d}.Wxa", [4 * H, H], s, trainable=True)
                Wb = g.placeholder(f"l{l}.{d}.Wxb", [4 * H, H], s, trainable=True)
            Wh = g.placeholder(f"l{l}.{d}.Wh", [4 * H, H], s, trainable=True)
            b = g.placeholder(f"l{l}.{d}.b", [4 * H], "f32", trainable=True)
            order = range(T) if d == "fw" else range(T - 1, -1, -1)
            h, c = h0, c0
            hs = [None] * T
            for t in order:
                if l == 0:
                    gx, extra = g.op("fully_connected", [xs[t], Wx, b], tag="rnn"), None
                else:
                    gx = g.op("fully_connected", [low["fw"][t], Wa, b], tag="rnn")
                    extra = g.op("fully_connected", [low["bw"][t], Wb], tag="rnn")
                h, c = lstm_cell(g, gx, h, c, Wh, H, B, s, tag="rnn", gh=True, extra=extra)
                hs[t] = h
            outs[d] = hs
        low = outs
    Woa = g.placeholder("out.Wa", [C, H], s, trainable=True)
    Wob = g.placeholder("out.Wb", [C, H], s, trainable=True)
    bo = g.placeholder("out.b", [C], "f32", trainable=True)
    logits = [g.op("add", [g.op("fully_connected", [low["fw"][t], Woa, bo], tag="output", dtype="f32"),
                           g.op("fully_connected", [low["bw"][t], Wob], tag="output", dtype="f32")], tag="output")
              for t in range(T)]
    loss, _ = g.op("softmax_ce_loss", [g.op("stack", logits, tag="output"), labels], tag="output", nout=2)
    g.output(loss)
    return g.doc()


def transformer(cfg, s="f32"):
    """Transformer attention-block stack with the op structure of the GPU path
    (paper_1805_08899_b200/transformer.py): per block q,k,v = FC(x); heads; S = batched_dot(qh, kh^T);
    P = softmax(S) (scale folded); (P_d, mask) = dropout(P); O = from_heads(batched_dot(P_d, vh));
    y = FC(O, Wo) + x.  Loss = sum(FC(y_final, r))."""
    B, L, d, H = cfg.B, cfg.L, cfg.d_model, cfg.heads
    N = B * L
    g = GraphBuilder()
    x = g.placeholder("x", [N, d], s)
    for k in range(cfg.blocks):
        W = {n: g.placeholder(f"b{k}.{n}", [d, d], s, trainable=True) for n in ("Wq", "Wk", "Wv", "Wo")}
        q, kk, v = (g.op("fully_connected", [x, W[n]], tag="tx") for n in ("Wq", "Wk", "Wv"))
        qh, kh, vh = (g.op("to_heads", [e], tag="tx", batch=B, heads=H) for e in (q, kk, v))
        S = g.op("batched_dot", [qh, kh], tag="attention", trans_b=1)
        P = g.op("softmax", [S], tag="attention")
        Pd, _mask = g.op("dropout", [P], tag="attention", nout=2, p=cfg.dropout_p)
        Oh = g.op("batched_dot", [Pd, vh], tag="attention")
        O = g.op("from_heads", [Oh], tag="tx", heads=H)
        x = g.op("add", [g.op("fully_connected", [O, W["Wo"]], tag="tx"), x], tag="tx")
    r = g.placeholder("out.r", [1, d], s, trainable=True)
    g.output(g.op("sum_reduce", [g.op("fully_connected", [x, r], tag="output")]))
    return g.doc()


# ----------------------------------------------------------------------------- random graphs
CHEAP_UNARY = ["tanh", "sigmoid", "relu"]
CHEAP_BINARY = ["add", "mul"]


CHEAP_UNARY_X = CHEAP_UNARY + ["gelu", "silu", "scale"]


def random_graph(seed, max_nodes=40, N=8, extended=False):
    """Seeded random DAG mixing cheap / compute-heavy / binarizable ops over [N, N] tensors.
    extended=True also draws the fx pass's gelu / silu / scale and 3-output layer_norm nodes."""
    rng = np.random.default_rng(seed)
    unary = CHEAP_UNARY_X if extended else CHEAP_UNARY
    g = GraphBuilder()
    edges = [g.placeholder(f"x{i}", [N, N], "f32") for i in range(int(rng.integers(1, 4)))]
    W = g.placeholder("W", [N, N], "f32", trainable=True)
    n_ops = int(rng.integers(3, max_nodes))
    for _ in range(n_ops):
        r = rng.random()
        a = edges[int(rng.integers(0, len(edges)))]
        if extended and r < 0.08:
            e = g.op("layer_norm", [a], nout=3, norm_ndim=1)[0]
        elif r < 0.35:
            e = g.op(unary[int(rng.integers(0, len(unary)))], [a])
        elif r < 0.65:
            b = edges[int(rng.integers(0, len(edges)))]
            e = g.op(CHEAP_BINARY[int(rng.integers(0, 2))], [a, b])
        elif r < 0.85:
            e = g.op("fully_connected", [a, W])
        else:
            e = g.op("dropout", [a], nout=2, p=0.5)[0]
        edges.append(e)
    # loss over the last few edges
    tail = edges[-int(rng.integers(1, min(4, len(edges)) + 1)):]
    loss = None
    for e in tail:
        s = g.op("sum_reduce", [e])
        loss = s if loss is None else g.op("add", [loss, s])
    g.output(loss)
    return g.doc()
