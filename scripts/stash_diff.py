import json, sys
sys.path.insert(0, '.')
import torch
from paper_1805_08899_b200 import abi
from paper_1805_08899_b200.nmt import NMTModel
from synth import graphs as Gr
from synth.configs import C1
from synth.data import nmt_batch
cfg = C1
for mode, strat in ((abi.STASH, "baseline"), (abi.RECOMPUTE, "echo")):
    rep = json.loads(abi.echo_footprint_estimate(json.dumps(Gr.nmt(cfg)), json.dumps({"strategy": strat})))
    m = NMTModel(cfg, abi.FP32, mode); m.upload_batch(nmt_batch(0, cfg)); acts = m._forward()
    print(strat, "gpu", m.stash_bytes(), "est", rep["stash_bytes"], rep["by_tag"])
    print({k: (tuple(v.shape), v.numel() * v.element_size(), v.data_ptr() % 100000) for k, v in m.stash.items()})
