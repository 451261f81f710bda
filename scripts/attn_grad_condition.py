"""Condition numbers of the attention-query gradients (diagnostic for reading R14b), oracle only (CPU).

For the bias b_q (folded into Kp, reading R3) the gradient is a plain sum over decoder steps t, rows b
and source positions s of dE_{t,b,s,a} = ds_{t,b,s} v_a (1 - E^2), with sum_s ds_{t,b,s} = 0 (softmax
backward): kappa = max_a sum|dE| / max_a |sum dE| measures the cancellation.  Likewise for v
(terms ds_{t,b,s} E_{t,b,s,a}).  A bf16-storage computation (unit roundoff u = 2^-8 on the stored
z = qp + Kp, E) is expected to reach an inf-norm relative error of order u * kappa.

Second check (emulate): the fp64 oracle step with the attention path's stored tensors rounded to bf16
as the GPU stores them (qp, Kp, H_s, and the feature map z = qp + Kp before the tanh; contract a4),
and the inf-norm relative change of the query-path gradients that this rounding alone causes.

usage: python scripts/attn_grad_condition.py
"""
import json
import os
import sys
import types

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from oracle import attention, nmt as ON  # noqa: E402
from synth.configs import SMALL_NMT, C2, NMTConfig  # noqa: E402
from synth import data as D  # noqa: E402

RAGGED = NMTConfig("ragged", B=5, Ts=11, Td=7, E=24, H=40, A=32, V=50, enc_layers=2, dec_layers=2)


def kappa(cfg, pseed, bseed):
    acc = {"bq_abs": 0.0, "bq": 0.0, "v_abs": 0.0, "v": 0.0}
    orig = attention.backward

    def wrapped(qp, Kp, v, Hs, dctx, src_len=None):
        r = orig(qp, Kp, v, Hs, dctx, src_len)
        dE, E = r["dKp"], r["E"]
        dalpha = np.einsum("bk,bsk->bs", np.asarray(dctx, np.float64), np.asarray(Hs, np.float64))
        al = r["alpha"]
        ds = al * (dalpha - (al * dalpha).sum(axis=1, keepdims=True))
        acc["bq_abs"] = acc["bq_abs"] + np.abs(dE).sum(axis=(0, 1))
        acc["bq"] = acc["bq"] + dE.sum(axis=(0, 1))
        acc["v_abs"] = acc["v_abs"] + np.einsum("bs,bsa->a", np.abs(ds), np.abs(E))
        acc["v"] = acc["v"] + r["dv"]
        return r
    attention.backward = wrapped
    try:
        ON.step(D.nmt_params(pseed, cfg, "bf16"), D.nmt_batch(bseed, cfg, lengths="random"), cfg)
    finally:
        attention.backward = orig
    return {k: float(np.max(acc[k + "_abs"]) / np.max(np.abs(acc[k]))) for k in ("bq", "v")}


def bf16(x):
    """round-to-nearest-even fp32 -> bf16, returned as float64"""
    a = np.asarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((a + 0x7FFF + ((a >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32).astype(np.float64)


def emulate(cfg, pseed, bseed):
    rel = lambda x, y: float(np.abs(x - y).max() / np.abs(y).max())
    P, B = D.nmt_params(pseed, cfg, "bf16"), D.nmt_batch(bseed, cfg, lengths="random")
    ref = ON.step(P, B, cfg)["grads"]
    shim = types.SimpleNamespace(**{k: getattr(np, k) for k in dir(np) if not k.startswith("__")})
    shim.tanh = lambda x: np.tanh(bf16(x))                 # attention.forward's only tanh: E = tanh(z)
    of, ob = attention.forward, attention.backward
    attention.np = shim
    attention.forward = lambda qp, Kp, v, Hs, src_len=None: of(bf16(qp), bf16(Kp), v, bf16(Hs), src_len)
    attention.backward = lambda qp, Kp, v, Hs, dctx, src_len=None: ob(bf16(qp), bf16(Kp), v, bf16(Hs), dctx, src_len)
    try:
        emu = ON.step(P, B, cfg)["grads"]
    finally:
        attention.np, attention.forward, attention.backward = np, of, ob
    return {k: rel(emu[k], ref[k]) for k in ("att.bq", "att.Wq", "att.v", "att.Wk")}


if __name__ == "__main__":
    u = 2.0 ** -8
    for cfg, seeds in ((SMALL_NMT, [(3, 4), (11, 12)]), (RAGGED, [(3, 4), (11, 12)]), (C2, [(3, 4)])):
        for ps, bs in seeds:
            k = kappa(cfg, ps, bs)
            print(json.dumps({"config": cfg.name, "seeds": [ps, bs], "kappa": k,
                              "u_kappa": {n: u * x for n, x in k.items()},
                              "stored_bf16_emulation_inf_relerr": emulate(cfg, ps, bs)}), flush=True)
