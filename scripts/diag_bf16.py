import sys, numpy as np, torch
sys.path.insert(0, '.')
torch.backends.cuda.matmul.allow_tf32 = False
from oracle import nmt as O
from synth.configs import C1, SMALL_NMT, NMTConfig
from synth.data import nmt_params, nmt_batch
from tests.gpu_util import relerr
from paper_1805_08899_b200 import abi
from paper_1805_08899_b200.nmt import NMTModel
RAGGED = NMTConfig("ragged", B=5, Ts=11, Td=7, E=24, H=40, A=32, V=50, enc_layers=2, dec_layers=2)
for cfg in (C1, SMALL_NMT, RAGGED):
    params = nmt_params(11, cfg, "bf16"); batch = nmt_batch(12, cfg, lengths="random")
    ref = O.step(params, batch, cfg)
    m = NMTModel(cfg, abi.BF16, abi.RECOMPUTE); m.load_params(params); m.upload_batch(batch)
    loss = m.train_step(lr=0.0); g = m.grads_numpy()
    errs = {k: relerr(g[k], v) for k, v in ref["grads"].items()}
    print(cfg.name, "loss", loss, ref["loss"], " worst:", sorted(errs.items(), key=lambda x: -x[1])[:6])
