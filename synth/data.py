"""Seeded input generators (numpy PCG64).  No method arithmetic lives here.

Recipe:
  * weights ~ U(-1/sqrt(H), +1/sqrt(H))  (the usual LSTM init)
  * embeddings, activations, upstream gradients ~ N(0, 1)
  * tokens ~ uniform over [0, V); source lengths full for throughput runs,
    uniform in [1, Ts] for parity runs
Every array is produced in float32 and, for bf16 storage, rounded to the
nearest bf16 value, so the GPU and the fp64 oracle consume identical numbers.
"""
from __future__ import annotations

import numpy as np

from .configs import NMTConfig, DS2Config


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def round_bf16(x: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bf16 (ties to even); returns float32."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    u = x.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def as_storage(x: np.ndarray, storage: str) -> np.ndarray:
    x = np.asarray(x, dtype=np.float32)
    if storage == "fp32":
        return x
    if storage == "bf16":
        return round_bf16(x)
    raise ValueError(storage)


def uniform(g, shape, bound):
    return g.uniform(-bound, bound, size=shape).astype(np.float32)


def normal(g, shape, scale=1.0):
    return (g.standard_normal(size=shape) * scale).astype(np.float32)


# ----------------------------------------------------------------------------- LSTM

def lstm_layer_inputs(seed, T, B, I, H, storage="fp32", state="random"):
    """One LSTM layer: X [T,B,I], Wx [4H,I], Wh [4H,H], b [4H] (fp32), h0, c0 [B,H], dH [T,B,H]."""
    g = rng(seed)
    k = 1.0 / np.sqrt(H)
    d = {
        "X": as_storage(normal(g, (T, B, I)), storage),
        "Wx": as_storage(uniform(g, (4 * H, I), k), storage),
        "Wh": as_storage(uniform(g, (4 * H, H), k), storage),
        "b": uniform(g, (4 * H,), k),                     # bias is fp32 in both storages (a4)
        "h0": as_storage(normal(g, (B, H), 0.5) if state == "random" else np.zeros((B, H), np.float32), storage),
        "c0": normal(g, (B, H), 0.5) if state == "random" else np.zeros((B, H), np.float32),
        "dH": normal(g, (T, B, H)),                        # upstream gradient, fp32 (a4)
        "dcT": normal(g, (B, H), 0.5) if state == "random" else np.zeros((B, H), np.float32),
    }
    return d


def lstm_cell_inputs(seed, B, H, storage="fp32", scale=1.0):
    """Single pointwise step: pre-activation A [B,4H], c_prev, dh, dc_carry."""
    g = rng(seed)
    return {
        "A": as_storage(normal(g, (B, 4 * H), scale), storage),
        "c_prev": normal(g, (B, H)),
        "dh": normal(g, (B, H)),
        "dc": normal(g, (B, H)),
    }


# ----------------------------------------------------------------------------- MLP attention

def mlp_attn_inputs(seed, B, Ts, A, Hk, storage="fp32", lengths="random"):
    """qp [B,A], Kp [B,Ts,A], v [A], Hs [B,Ts,Hk], src_len [B] int32, dctx [B,Hk]."""
    g = rng(seed)
    if lengths == "full":
        src_len = np.full((B,), Ts, np.int32)
    else:
        src_len = g.integers(1, Ts + 1, size=(B,)).astype(np.int32)
        src_len[0] = Ts  # always exercise a full row
    return {
        "qp": as_storage(normal(g, (B, A), 0.5), storage),
        "Kp": as_storage(normal(g, (B, Ts, A), 0.5), storage),
        "v": as_storage(uniform(g, (A,), 1.0 / np.sqrt(A)) * 4.0, storage),
        "Hs": as_storage(normal(g, (B, Ts, Hk)), storage),
        "src_len": src_len,
        "dctx": normal(g, (B, Hk)),
    }


# ----------------------------------------------------------------------------- dot softmax + dropout

def dot_softmax_inputs(seed, R, L, storage="fp32"):
    """Scores S [R,L] (as produced by the caller's QK^T GEMM) and upstream dPd [R,L]."""
    g = rng(seed)
    return {
        "S": as_storage(normal(g, (R, L), 2.0), storage),
        "dPd": as_storage(normal(g, (R, L)), storage),
    }


# ----------------------------------------------------------------------------- NMT model

def nmt_param_shapes(cfg: NMTConfig):
    """Ordered (name, shape) list of every trainable tensor of the NMT model.

    Structure only (§2 Fig. 2; readings R3, R7 in DESIGN.md):
      encoder LSTM layers, decoder LSTM layers with input feeding (layer-0 input
      is [emb(y_{t-1}); a_{t-1}]), MLP attention (W_q, b_q, W_k, v), attention
      hidden a_t = tanh(W_cc ctx + W_ch h), output FC W_o, b_o.
    """
    H, E, A, V = cfg.H, cfg.E, cfg.A, cfg.V
    shapes = [("emb_src", (V, E)), ("emb_tgt", (V, E))]
    for l in range(cfg.enc_layers):
        I = E if l == 0 else H
        shapes += [(f"enc{l}.Wx", (4 * H, I)), (f"enc{l}.Wh", (4 * H, H)), (f"enc{l}.b", (4 * H,))]
    for l in range(cfg.dec_layers):
        I = E + H if l == 0 else H
        shapes += [(f"dec{l}.Wx", (4 * H, I)), (f"dec{l}.Wh", (4 * H, H)), (f"dec{l}.b", (4 * H,))]
    shapes += [("att.Wq", (A, H)), ("att.bq", (A,)), ("att.Wk", (A, cfg.Hk)), ("att.v", (A,)),
               ("att.Wcc", (H, cfg.Hk)), ("att.Wch", (H, H)),
               ("out.Wo", (V, H)), ("out.bo", (V,))]
    return shapes


def nmt_params(seed, cfg: NMTConfig, storage="fp32"):
    g = rng(seed)
    k = 1.0 / np.sqrt(cfg.H)
    out = {}
    for name, shape in nmt_param_shapes(cfg):
        if name.startswith("emb"):
            out[name] = as_storage(normal(g, shape), storage)
        elif name.endswith(".b") or name.endswith(".bq") or name.endswith(".bo"):
            out[name] = uniform(g, shape, k)                # biases fp32 (a4)
        else:
            out[name] = as_storage(uniform(g, shape, k), storage)
    return out


def nmt_batch(seed, cfg: NMTConfig, lengths="full"):
    """src [B,Ts], tgt_in [B,Td], tgt_out [B,Td] int64 tokens; src_len [B] int32."""
    g = rng(seed)
    src = g.integers(0, cfg.V, size=(cfg.B, cfg.Ts)).astype(np.int64)
    tgt = g.integers(0, cfg.V, size=(cfg.B, cfg.Td + 1)).astype(np.int64)
    if lengths == "full":
        src_len = np.full((cfg.B,), cfg.Ts, np.int32)
    else:
        src_len = g.integers(1, cfg.Ts + 1, size=(cfg.B,)).astype(np.int32)
        src_len[0] = cfg.Ts
    # Philox keys of the two embedding-dropout sites (source, target), drawn per batch (R31)
    seeds = g.integers(1, 2 ** 62, size=2).astype(np.uint64)
    nh = cfg.hidden_drop_sites()
    if nh:                                                   # reading R33: one key per hidden site, after
        seeds = np.concatenate([seeds, g.integers(1, 2 ** 62, size=nh).astype(np.uint64)])   # the two above
    return {"src": src, "tgt_in": tgt[:, :-1].copy(), "tgt_out": tgt[:, 1:].copy(), "src_len": src_len,
            "drop_seeds": seeds}


# ----------------------------------------------------------------------------- DS2

def ds2_param_shapes(cfg: DS2Config):
    shapes = []
    for l in range(cfg.layers):
        I = cfg.F if l == 0 else 2 * cfg.H
        for d in ("fw", "bw"):
            shapes += [(f"l{l}.{d}.Wx", (4 * cfg.H, I)), (f"l{l}.{d}.Wh", (4 * cfg.H, cfg.H)),
                       (f"l{l}.{d}.b", (4 * cfg.H,))]
    shapes += [("out.W", (cfg.classes, 2 * cfg.H)), ("out.b", (cfg.classes,))]
    return shapes


def ds2_params(seed, cfg: DS2Config, storage="fp32"):
    g = rng(seed)
    k = 1.0 / np.sqrt(cfg.H)
    out = {}
    for name, shape in ds2_param_shapes(cfg):
        if name.endswith(".b"):
            out[name] = uniform(g, shape, k)
        else:
            out[name] = as_storage(uniform(g, shape, k), storage)
    return out


def ds2_batch(seed, cfg: DS2Config, storage="fp32"):
    g = rng(seed)
    return {"x": as_storage(normal(g, (cfg.T, cfg.B, cfg.F)), storage),
            "labels": g.integers(0, cfg.classes, size=(cfg.T, cfg.B)).astype(np.int64)}


# ----------------------------------------------------------------------------- Transformer attention blocks
def tx_param_shapes(cfg):
    d = cfg.d_model
    shapes = []
    for k in range(cfg.blocks):
        shapes += [(f"b{k}.Wq", (d, d)), (f"b{k}.Wk", (d, d)), (f"b{k}.Wv", (d, d)), (f"b{k}.Wo", (d, d))]
    shapes += [("out.r", (d,))]
    return shapes


def tx_params(seed, cfg, storage="fp32"):
    g = rng(seed)
    k = 1.0 / np.sqrt(cfg.d_model)
    return {name: as_storage(uniform(g, shape, k) if name != "out.r" else normal(g, shape), storage)
            for name, shape in tx_param_shapes(cfg)}


def tx_batch(seed, cfg, storage="fp32"):
    """x [B, L, d] ~ N(0,1); per-block dropout seeds."""
    g = rng(seed)
    return {"x": as_storage(normal(g, (cfg.B, cfg.L, cfg.d_model)), storage),
            "seeds": [int(s) for s in g.integers(1, 2 ** 40, size=cfg.blocks)]}
