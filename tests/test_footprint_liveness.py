"""Hand-counted pins for the estimator's liveness / peak model (oracle/footprint.py `schedule` +
`live_timeline`, and the C++ planner behind echo_footprint_estimate).

The numbers below were counted by hand from the liveness rules (R16), NOT produced by
either implementation.  The rules, restated:
  * schedule: every forward node in id (= topological) order; then, for each node in reverse id
    order, the mirror nodes its gradient needs (recursively, in id order) followed by its gradient.
  * a forward output lives from its producing step to its last reader: forward readers, plus --
    if it is kept across the forward -> backward boundary (stashed) -- the gradient steps and
    mirror steps that read it.  Placeholders (inputs, weights, c0/h0) are not activations.
  * a recomputed (mirror) output lives from its mirror step to its last reader in the backward.
  * the gradient of a float activation lives from the first gradient step that produces it (the
    earliest-scheduled consumer gradient; for the graph output, the first backward step) to the
    gradient step of its producer.
Paper passages: Alg. 1 decides the kept set; Fig. 4, Fig. 6/9
 are the worked examples.  A shifted lifetime (e.g. a gradient that lives
one step longer, a stashed edge freed at its last forward reader) changes at least one entry below.
"""
import json

import pytest

from oracle import footprint as F
from synth import graphs as Gr


@pytest.fixture(scope="module")
def est():
    from paper_1805_08899_b200 import build, abi
    build.build()
    abi.load()

    def run(doc, cfg=None):
        return json.loads(abi.echo_footprint_estimate(json.dumps(doc), json.dumps(cfg) if cfg is not None else None))
    return run


def _both(est, doc, strategy):
    o = F.analyze(doc, {"strategy": strategy})
    c = est(doc, {"strategy": strategy})
    return o["timeline"], c["timeline"], c["peak_bytes"]


# --------------------------------------------------------------------------- Fig. 6: Z = tanh(X + Y)
def test_add_tanh_timeline_hand_counted(est):
    """N = 1024 f32, one tensor = n = 4096 B; the scalar loss L and its gradient are 4 B.
    Nodes: a = add(X, Y) (id 2), Z = tanh(a) (3), L = sum(Z) (4).

    Baseline / Echo (Z kept for tanh's gradient, no mirrors) -- steps:
      0 fwd add: a                      = n
      1 fwd tanh: a (read now), Z       = 2n
      2 fwd sum: Z (kept), L            = n + 4
      3 grad sum: Z, dL, dZ             = 2n + 4
      4 grad tanh: Z (read), dZ, da     = 3n
      5 grad add: da                    = n
    Mirror (add and tanh mirrored; X, Y kept): Z is freed after the sum at step 2 --
      0 a = n; 1 a, Z = 2n; 2 Z, L = n + 4; 3 grad sum: dL, dZ = n + 4;
      4 mirror add: dZ, a' = 2n; 5 mirror tanh: dZ, a', Z' = 3n;
      6 grad tanh: dZ, Z', da = 3n; 7 grad add: da = n."""
    n = 1024 * 4
    doc = Gr.add_tanh(1024)
    base = [n, 2 * n, n + 4, 2 * n + 4, 3 * n, n]
    mirror = [n, 2 * n, n + 4, n + 4, 2 * n, 3 * n, 3 * n, n]
    for strategy, want in (("baseline", base), ("echo", base), ("mirror", mirror)):
        o, c, peak = _both(est, doc, strategy)
        assert o == want, (strategy, o)
        assert c == want, (strategy, c)
        assert peak == 3 * n


# --------------------------------------------------------------------------- Fig. 4: tanh chain
def test_chain4_timeline_hand_counted(est):
    """x -> t1 -> t2 -> t3 -> t4 -> sum, N = 64 f32: one edge = u = 256 B, L / dL = 4 B.

    Baseline keeps e1..e4 (each tanh's gradient reads its output):
      fwd  0: e1 | 1: e1 e2 | 2: e1-e3 | 3: e1-e4 | 4: e1-e4 L
      bwd  5 grad sum: e1-e4 dL de4 (5u+4) | 6 grad t4: e1-e4 de4 de3 (6u)
           7 grad t3: e1-e3 de3 de2 (5u) | 8 grad t2: e1 e2 de2 de1 (4u) | 9 grad t1: e1 de1 (2u)
    Echo keeps e1 only (t2..t4 mirrored; Fig. 4's one edge at the head of the chain):
      fwd  0: e1 | 1: e1 e2 | 2: e1 e2 e3 | 3: e1 e3 e4 (e2 freed) | 4: e1 e4 L
      bwd  5 grad sum: e1 dL de4 | 6-8 mirrors t2 t3 t4: + e2' + e3' + e4'
           9 grad t4: e1 e2' e3' e4' de4 de3 (6u) | 10 grad t3: e1 e2' e3' de3 de2 (5u)
           11 grad t2: e1 e2' de2 de1 (4u) | 12 grad t1: e1 de1 (2u)
    Mirror keeps only the input x (t1..t4 mirrored, e1 freed in the forward too):
      fwd  0: e1 | 1: e1 e2 | 2: e2 e3 | 3: e3 e4 | 4: e4 L
      bwd  5 grad sum: dL de4 | 6-9 mirrors t1..t4: de4 + e1' .. e4'
           10 grad t4: e1'-e4' de4 de3 (6u) | 11: e1'-e3' de3 de2 | 12: e1' e2' de2 de1 | 13: e1' de1"""
    u = 64 * 4
    doc = Gr.chain4(64)
    base = [u, 2 * u, 3 * u, 4 * u, 4 * u + 4, 5 * u + 4, 6 * u, 5 * u, 4 * u, 2 * u]
    echo = [u, 2 * u, 3 * u, 3 * u, 2 * u + 4, 2 * u + 4, 3 * u, 4 * u, 5 * u, 6 * u, 5 * u, 4 * u, 2 * u]
    mirror = [u, 2 * u, 2 * u, 2 * u, u + 4, u + 4, 2 * u, 3 * u, 4 * u, 5 * u, 6 * u, 5 * u, 4 * u, 2 * u]
    for strategy, want in (("baseline", base), ("echo", echo), ("mirror", mirror)):
        o, c, peak = _both(est, doc, strategy)
        assert o == want, (strategy, o)
        assert c == want, (strategy, c)
        assert peak == 6 * u


# --------------------------------------------------------------------------- T = 2 LSTM layer
def test_lstm_layer_t2_peak_hand_counted(est):
    """Gr.lstm_layer(T=2, B=2, H=8, I=8) f32: one [B,H] tensor = u = 64 B; [B,4H] = 4u; the
    per-step loss terms are scalars (4 B).  Node ids: step 0 -- gx0 6, gh0 7, A0 8, slices 9-12,
    gates i f g o 13-16, f*c0 17, i*g 18, c1 19, tanh c1 20, h1 21, FC(h1, Wo0) 23, sum0 24;
    step 1 -- gx1 26, gh1 27, A1 28, slices 29-32, gates 33-36, 37, 38, c2 39, tc2 40, h2 41, 43, 44,
    loss add 45.  37 forward steps, so the first backward step is 37.

    Baseline peak = 19u + 4 = 1220 B, first reached at step 20 (forward of A1 = gx1 + gh1).  Live:
      kept step-0 gates 13-16 (4u), c1 (u, read by mul 37's gradient), tanh c1 (u), h1 (u);
      sum0 (4 B, read by the loss add at step 36); gx1 (4u) and gh1 (4u) being read; A1 (4u).

    Echo mirrors {17-21, 37-41} (the c-chain, tanh c and h; the FCs reading h become dead
    mirrors), keeps the gates.  Peak = 18u + 4 = 1156 B at step 61 (gradient of A1 = add 28).  Live:
      kept step-0 gates 13-16 (4u; the step-1 gates were freed at their own gradients, 53-56);
      recomputed c1' (u: mirrored at 41, read by mirror tanh 20 at step 62);
      dA1 (4u, from slice 32's gradient at 57 to 61); dgx1 and dgh1 (4u each, produced here);
      dc1 (u, produced by mul 37's gradient at 52, consumed at add 19's gradient);
      dsum0 (4 B, produced at the first backward step 37, consumed at 66)."""
    u = 2 * 8 * 4
    doc = Gr.lstm_layer(2, 2, 8, 8)
    for strategy, peak, at in (("baseline", 19 * u + 4, 20), ("echo", 18 * u + 4, 61)):
        o, c, cpeak = _both(est, doc, strategy)
        assert max(o) == peak and o.index(peak) == at, (strategy, max(o), o.index(max(o)))
        assert c == o and cpeak == peak, strategy
    o = F.analyze(doc, {"strategy": "echo"})
    assert sorted(o["mirrored"]) == [17, 18, 19, 20, 21, 37, 38, 39, 40, 41]
    assert sorted(o["dead"]) == [23, 27, 43]
