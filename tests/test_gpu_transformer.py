"""Transformer attention blocks (a7 + cuBLAS) vs the fp64 oracle; STASH == RECOMPUTE bit-identity;
GPU stash bytes == estimator (Baseline / Echo / Mirror plans)."""
import json
from dataclasses import replace

import numpy as np
import pytest
import torch

from oracle import transformer as O
from synth.configs import SMALL_TX, C4
from synth.data import tx_params, tx_batch
from tests.gpu_util import relerr, bits_equal, check_grads

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _strict_fp32():
    torch.backends.cuda.matmul.allow_tf32 = False


def _run(cfg, params, batch, dtype, mode, mirror=False, regen=False):
    from paper_1805_08899_b200.transformer import TXModel
    m = TXModel(cfg, dtype, mode, mirror=mirror, regen_masks=regen)
    m.load_params(params)
    m.upload_batch(batch)
    return m, m.train_step(lr=0.0)


# bf16 storage: tensors gated on the Frobenius relative error (reading R14b); the rest on the inf-norm.
FRO_ONLY = {}


@pytest.mark.parametrize("cfg,storage", [(SMALL_TX, "fp32"), (SMALL_TX, "bf16"), (replace(C4, blocks=2), "fp32"),
                                         (replace(C4, blocks=2), "bf16")],
                         ids=["small-fp32", "small-bf16", "C4x2-fp32", "C4x2-bf16"])
def test_tx_parity_and_bit_identity(cfg, storage, cuda_dev):
    from paper_1805_08899_b200 import abi
    params = tx_params(1, cfg, storage)
    batch = tx_batch(2, cfg, storage)
    ref = O.step(params, batch, cfg)
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    tol = 1e-4 if storage == "fp32" else 2e-2
    res = {}
    plans = ((abi.STASH, False, False), (abi.RECOMPUTE, False, False), (abi.RECOMPUTE, True, False),
             (abi.RECOMPUTE, False, True), (abi.RECOMPUTE, True, True))
    for mode, mirror, regen in plans:
        m, loss = _run(cfg, params, batch, dt, mode, mirror, regen)
        assert abs(loss - ref["loss"]) <= tol * max(abs(ref["loss"]), 1e-3), (loss, ref["loss"])
        g = m.grads_numpy()
        check_grads(g, ref["grads"], storage, FRO_ONLY.get((cfg.name, cfg.blocks, storage), ()),
                    f"{cfg.name}/{mode}/{mirror}/{regen}")
        res[(mode, mirror, regen)] = m.gflat.clone()
    for p in plans[1:]:               # Echo, Mirror, and both with regenerated masks: the same gradients
        assert bits_equal(res[plans[0]], res[p]), p


@pytest.mark.parametrize("cfg", [SMALL_TX, C4], ids=lambda c: c.name)
@pytest.mark.parametrize("storage", ["fp32", "bf16"])
def test_tx_stash_bytes_equal_estimator(cfg, storage, cuda_dev):
    from paper_1805_08899_b200 import abi
    from paper_1805_08899_b200.transformer import TXModel
    from synth import graphs as Gr
    doc = json.dumps(Gr.transformer(cfg, "f32" if storage == "fp32" else "bf16"))
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    for mode, strat, regen in ((abi.STASH, "baseline", False), (abi.RECOMPUTE, "echo", False),
                               (abi.RECOMPUTE, "mirror", False), (abi.RECOMPUTE, "echo", True),
                               (abi.RECOMPUTE, "mirror", True)):
        rep = json.loads(abi.echo_footprint_estimate(doc, json.dumps({"strategy": strat, "regenerate_masks": regen})))
        m = TXModel(cfg, dt, mode, mirror=strat == "mirror", regen_masks=regen)
        m.upload_batch(tx_batch(0, cfg, storage))
        acts = m._forward()
        assert m.stash_bytes() == rep["stash_bytes"], (strat, m.stash_bytes(), rep["stash_bytes"])
        del acts


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
def test_tx_c4_full_bitwise_and_graph(storage, cuda_dev):
    """Full C4 (6 blocks, B=64, L=256, d=512, 8 heads, dropout 0.1): STASH == RECOMPUTE bitwise and
    graph replay == eager bitwise."""
    from paper_1805_08899_b200 import abi
    params = tx_params(3, C4, storage)
    batch = tx_batch(4, C4, storage)
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    res = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        m, loss = _run(C4, params, batch, dt, mode)
        res[mode] = (m.gflat.clone(), m.loss.clone())
        if mode == abi.RECOMPUTE:
            m.capture(0.0)
            m.gflat.zero_()
            m.replay()
            torch.cuda.synchronize()
            assert bits_equal(m.gflat, res[mode][0])
        del m
        torch.cuda.empty_cache()
    assert bits_equal(res[abi.STASH][0], res[abi.RECOMPUTE][0])
    assert bits_equal(res[abi.STASH][1], res[abi.RECOMPUTE][1])
