"""a1 / a2 / a3 vector width (ECHO_LSTM_VEC): every width gives bit-identical outputs (the per-element
arithmetic does not depend on how many elements a thread owns).  Each width runs in its own
process because the library reads the variable once."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
from paper_1805_08899_b200 import abi
from synth.data import lstm_cell_inputs
abi.load()
storage, mode, out = sys.argv[2], sys.argv[3], sys.argv[4]
B, H = 96, 520
d = lstm_cell_inputs(5, B, H, storage)
sd = torch.float32 if storage == "fp32" else torch.bfloat16
dt = abi.FP32 if storage == "fp32" else abi.BF16
m = abi.STASH if mode == "stash" else abi.RECOMPUTE
desc = abi.LstmDesc(B, H, dt, m)
A = torch.from_numpy(np.asarray(d["A"], np.float32)).cuda().to(sd)
gh = torch.from_numpy(np.asarray(d["A"], np.float32)[::-1].copy()).cuda().to(sd) * 0.5
bias = torch.linspace(-1, 1, 4 * H, device="cuda")
cp = torch.from_numpy(np.asarray(d["c_prev"], np.float32)).cuda()
gates = torch.empty_like(A); c = torch.empty(B, H, device="cuda")
tc = torch.empty(B, H, device="cuda", dtype=sd) if m == abi.STASH else None
h = torch.empty(B, H, device="cuda", dtype=sd)
abi.echo_lstm_fwd(desc, A, gh, bias, cp, gates, c, tc, h)
dh = torch.from_numpy(np.asarray(d["dh"], np.float32)).cuda()
dc = torch.from_numpy(np.asarray(d["dc"], np.float32)).cuda()
dA = torch.empty_like(A)
hreg = torch.empty_like(h) if m == abi.RECOMPUTE else None
if m == abi.STASH:
    abi.echo_lstm_bwd_recompute(desc, 1, 0, 0, gates, cp, None, tc, dh, dc, dA, None, None)
else:
    abi.echo_lstm_bwd_recompute(desc, 1, 0, 0, gates, cp, None, None, dh, dc, dA, hreg, c)
T = 7
G = torch.rand(T, B, 4 * H, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3)).to(sd)
cws = torch.empty(T, B, H, device="cuda"); hws = torch.empty(T, B, H, device="cuda", dtype=sd)
abi.echo_lstm_cscan(abi.LstmDesc(B, H, dt, abi.RECOMPUTE), T, G, cp, cws, hws)
torch.cuda.synchronize()
res = {"cws": cws, "hws": hws, "gates": gates, "c": c, "h": h, "dA": dA, "dc": dc}
if hreg is not None: res["hreg"] = hreg
if tc is not None: res["tc"] = tc
np.savez(out, **{k: v.contiguous().view(torch.int16 if v.dtype == torch.bfloat16 else torch.int32).cpu().numpy()
                 for k, v in res.items()})
"""


@pytest.mark.parametrize("storage,widths", [("fp32", [1, 2, 4]), ("bf16", [2, 4, 8])])
@pytest.mark.parametrize("mode", ["stash", "recompute"])
def test_vector_width_bit_identical(storage, widths, mode, tmp_path):
    outs = []
    for v in widths:
        out = str(tmp_path / f"v{v}.npz")
        env = dict(os.environ, ECHO_LSTM_VEC=str(v))
        r = subprocess.run([sys.executable, "-c", CHILD, ROOT, storage, mode, out], env=env, capture_output=True,
                           text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(out))
    for k in outs[0].files:
        for v, o in zip(widths[1:], outs[1:]):
            assert np.array_equal(outs[0][k], o[k]), f"{k}: width {v} differs from width {widths[0]}"
