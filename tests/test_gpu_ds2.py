"""DeepSpeech2-shaped bidirectional LSTM stack on the GPU vs the fp64 oracle; STASH == RECOMPUTE
bit-identity; GPU stash bytes == estimator."""
import json
from dataclasses import replace

import pytest
import torch

from oracle import ds2 as O
from synth.configs import SMALL_DS2, C3
from synth.data import ds2_params, ds2_batch
from tests.gpu_util import relerr, relerr_fro, bits_equal

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _strict_fp32():
    torch.backends.cuda.matmul.allow_tf32 = False


@pytest.mark.parametrize("cfg,storage", [(SMALL_DS2, "fp32"), (SMALL_DS2, "bf16"), (replace(C3, layers=2), "fp32")],
                         ids=["small-fp32", "small-bf16", "C3x2-fp32"])
def test_ds2_parity_and_bit_identity(cfg, storage, cuda_dev):
    from paper_1805_08899_b200 import abi
    from paper_1805_08899_b200.ds2 import DS2Model
    params = ds2_params(1, cfg, storage)
    batch = ds2_batch(2, cfg, storage)
    ref = O.step(params, batch, cfg)
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    tol = 1e-4 if storage == "fp32" else 2e-2
    metric = relerr if storage == "fp32" else relerr_fro
    res = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        m = DS2Model(cfg, dt, mode)
        m.load_params(params)
        m.upload_batch(batch)
        loss = m.train_step(lr=0.0)
        assert abs(loss - ref["loss"]) <= tol * abs(ref["loss"]), (loss, ref["loss"])
        g = m.grads_numpy()
        for k, v in ref["grads"].items():
            assert metric(g[k], v) <= tol, (k, metric(g[k], v))
        res[mode] = m.gflat.clone()
    assert bits_equal(res[abi.STASH], res[abi.RECOMPUTE])


@pytest.mark.parametrize("cfg", [SMALL_DS2, C3], ids=lambda c: c.name)
@pytest.mark.parametrize("storage", ["fp32", "bf16"])
def test_ds2_stash_bytes_equal_estimator(cfg, storage, cuda_dev):
    from paper_1805_08899_b200 import abi
    from paper_1805_08899_b200.ds2 import DS2Model
    from synth import graphs as Gr
    doc = json.dumps(Gr.ds2(cfg, "f32" if storage == "fp32" else "bf16"))
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    for mode, strat in ((abi.STASH, "baseline"), (abi.RECOMPUTE, "echo")):
        rep = json.loads(abi.echo_footprint_estimate(doc, json.dumps({"strategy": strat})))
        m = DS2Model(cfg, dt, mode)
        acts = m._forward()
        assert m.stash_bytes() == rep["stash_bytes"], (strat, m.stash_bytes(), rep["stash_bytes"])
        del acts


@pytest.mark.parametrize("storage", ["fp32", "bf16"])
def test_ds2_c3_full_bitwise_and_graph(storage, cuda_dev):
    """Full C3 (5 bidirectional layers, T=400, B=32, H=800) in the bench launch configuration:
    STASH == RECOMPUTE bitwise (loss and every gradient), and the CUDA-graph replay (the two
    directions as parallel branches) == the eager step bitwise."""
    from paper_1805_08899_b200 import abi
    from paper_1805_08899_b200.ds2 import DS2Model
    params = ds2_params(7, C3, storage)
    batch = ds2_batch(8, C3, storage)
    dt = abi.FP32 if storage == "fp32" else abi.BF16
    res = {}
    for mode in (abi.STASH, abi.RECOMPUTE):
        m = DS2Model(C3, dt, mode)
        m.load_params(params)
        m.upload_batch(batch)
        m.step(0.0)
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
    assert torch.isfinite(res[abi.STASH][0]).all()
