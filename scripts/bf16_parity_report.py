"""bf16-storage parity report (diagnostic for reading R14b): for every bf16 model configuration, the
per-tensor max relative error (inf-norm, north_star's metric) and the Frobenius relative error of the
GPU gradients against the fp64 oracle, next to the tensor's bf16 NOISE FLOOR: the inf-norm relative
change of the ORACLE's own gradient when every parameter and input is perturbed by a relative
2^-9 N(0,1) (the size of one bf16 rounding).  A tensor whose floor is itself ~2e-2 cannot meet the
inf-norm bound in any bf16-storage implementation (cancellation-dominated sums); the GPU error
should be a small multiple of the floor.

usage: python scripts/bf16_parity_report.py [--configs small,ragged,c2,ds2s,c3x2,txs,c4x2] > report.json
"""
import argparse
import json
import os
import sys
from dataclasses import replace

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from synth.configs import SMALL_NMT, C2, C3, C4, SMALL_DS2, SMALL_TX, NMTConfig  # noqa: E402
from synth import data as D  # noqa: E402

RAGGED = NMTConfig("ragged", B=5, Ts=11, Td=7, E=24, H=40, A=32, V=50, enc_layers=2, dec_layers=2)


def relerr(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    d = np.abs(y).max()
    return float(np.abs(x - y).max() / (d if d > 0 else 1.0))


def fro(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    d = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / (d if d > 0 else 1.0))


def perturb(tree, g):
    out = {}
    for k, v in tree.items():
        if isinstance(v, np.ndarray) and v.dtype.kind == "f":
            out[k] = v * (1.0 + 2.0 ** -9 * g.standard_normal(v.shape))
        else:
            out[k] = v
    return out


def case(name):
    from paper_1805_08899_b200 import abi
    from oracle import nmt as ON, ds2 as OD, transformer as OT
    if name in ("small", "ragged", "c2"):
        from paper_1805_08899_b200.nmt import NMTModel
        cfg = {"small": SMALL_NMT, "ragged": RAGGED, "c2": C2}[name]
        P, B = D.nmt_params(3, cfg, "bf16"), D.nmt_batch(4, cfg, lengths="random")
        run_o = lambda P, B: ON.step(P, B, cfg)
        m = NMTModel(cfg, dtype=abi.BF16, mode=abi.RECOMPUTE)
        m.load_params(P)
        m.upload_batch(B)
        m.train_step(lr=0.0)
    elif name in ("ds2s", "c3x2"):
        from paper_1805_08899_b200.ds2 import DS2Model
        cfg = SMALL_DS2 if name == "ds2s" else replace(C3, layers=2)
        P, B = D.ds2_params(1, cfg, "bf16"), D.ds2_batch(2, cfg, "bf16")
        run_o = lambda P, B: OD.step(P, B, cfg)
        m = DS2Model(cfg, abi.BF16, abi.RECOMPUTE)
        m.load_params(P)
        m.upload_batch(B)
        m.train_step(lr=0.0)
    else:
        from paper_1805_08899_b200.transformer import TXModel
        cfg = SMALL_TX if name == "txs" else replace(C4, blocks=2)
        P, B = D.tx_params(1, cfg, "bf16"), D.tx_batch(2, cfg, "bf16")
        keep = OT.masks(cfg, B["seeds"])
        run_o = lambda P, B: OT.step(P, B, cfg, keep)
        m = TXModel(cfg, abi.BF16, abi.RECOMPUTE)
        m.load_params(P)
        m.upload_batch(B)
        m.train_step(lr=0.0)
    g = m.grads_numpy()
    ref = run_o(P, B)
    gen = np.random.default_rng(0)
    pref = run_o(perturb({k: np.asarray(v, np.float64) for k, v in P.items()}, gen), perturb(dict(B), gen))
    rows = {}
    for k, v in ref["grads"].items():
        rows[k] = {"inf": relerr(g[k], v), "fro": fro(g[k], v), "floor_inf": relerr(pref["grads"][k], v),
                   "floor_fro": fro(pref["grads"][k], v)}
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="small,ragged,ds2s,txs,c3x2,c4x2,c2")
    a = ap.parse_args()
    torch.backends.cuda.matmul.allow_tf32 = False
    from paper_1805_08899_b200 import abi
    abi.load()
    for name in a.configs.split(","):
        rows = case(name)
        bad = {k: r for k, r in rows.items() if r["inf"] > 2e-2}
        print(json.dumps({"config": name, "max_inf": max(r["inf"] for r in rows.values()),
                          "over_2e-2": bad, "all": rows}), flush=True)


if __name__ == "__main__":
    main()
