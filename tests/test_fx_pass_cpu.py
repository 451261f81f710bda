"""The automatic fx pass on the host: tracing into the estimator's schema, the
plan's decisions, and refusals (no GPU needed; the GPU run is tests/test_gpu_fx_pass.py)."""
import json

import pytest
import torch
import torch.nn as nn

from tests.fx_models import GatedNet, ResMLP, ReluTaps, ResConvNet


@pytest.fixture(scope="module", autouse=True)
def _lib():
    from paper_1805_08899_b200 import build, abi
    build.build()
    abi.load()


def test_plan_of_gated_net():
    from paper_1805_08899_b200 import fx_pass as X
    m = GatedNet(16, 2)
    x = torch.randn(8, 16)
    p = X.EchoPlan(m, (x,))
    ops = [n["op"] for n in p.doc["nodes"]]
    assert ops.count("fully_connected") == 7 and ops.count("dropout") == 2 and ops.count("mul") == 2
    assert sum(1 for q in p.doc["placeholders"] if q["trainable"]) == 14          # 7 weights + 7 biases
    b = X.EchoPlan(m, (x,), strategy="baseline")
    assert p.stash_bytes() < b.stash_bytes()
    kinds = set(p.decision.values())
    assert "recompute" in kinds and "bit" in kinds                # mirrored maps and 1-bit dropout masks
    # the plan is the estimator's: the same document through the C ABI gives the same bytes
    from paper_1805_08899_b200 import abi
    r = json.loads(abi.echo_footprint_estimate(json.dumps(p.doc), json.dumps({"strategy": "echo"})))
    assert r["stash_bytes"] == p.stash_bytes()


def test_plan_recomputes_relu_maps():
    """ReLU outputs between FCs: Echo keeps the FC outputs the FCs need anyway and regenerates the ReLU
    maps (mirrored, Fig. 4) instead of keeping them -- here better than 1-bit signs (0 extra bytes);
    never worse than the Baseline on a residual MLP either."""
    from paper_1805_08899_b200 import fx_pass as X
    m = ReluTaps(16, 3)
    x = torch.randn(4, 16)
    p = X.EchoPlan(m, (x,))
    b = X.EchoPlan(m, (x,), strategy="baseline")
    relu_ids = [n["id"] for n in p.doc["nodes"] if n["op"] == "relu"]
    assert all(p.decision.get((i, 0)) == "recompute" for i in relu_ids)
    assert all(b.decision.get((i, 0)) == "stash" for i in relu_ids if (i, 0) in b.decision)
    assert b.stash_bytes() - p.stash_bytes() == 2 * 4 * 16 * 4
    r = ResMLP(16, 3)
    assert X.EchoPlan(r, (x,)).stash_bytes() <= X.EchoPlan(r, (x,), strategy="baseline").stash_bytes()


def test_unsupported_ops_raise():
    from paper_1805_08899_b200 import fx_pass as X

    class Conv(nn.Module):
        def __init__(self):
            super().__init__()
            self.c = nn.Conv1d(2, 2, 3)

        def forward(self, x):
            return self.c(x).sum()

    class Bcast(nn.Module):
        def forward(self, x):
            return (x + x[:1]).sum()
    with pytest.raises(X.Unsupported):
        X.EchoPlan(Conv(), (torch.randn(1, 2, 8),))
    with pytest.raises(X.Unsupported):
        X.EchoPlan(Bcast(), (torch.randn(4, 8),))


def test_conv2d_graph_cpp_equals_oracle():
    """conv2d (compute-heavy, its gradient reads input and weight): the traced ResNet-style CNN through
    the C++ estimator equals the Python oracle (bytes, timeline, recompute flops) for every plan; Echo
    never keeps more than the Baseline; the unmodified model's autograd keeps exactly the Baseline bytes."""
    from oracle import footprint as F
    from paper_1805_08899_b200 import fx_pass as X
    m = ResConvNet(8, 2)
    x = torch.randn(2, 3, 16, 16)
    for st in ("baseline", "echo", "mirror"):
        p = X.EchoPlan(m, (x,), strategy=st)
        o = F.analyze(p.doc, {"strategy": st})
        assert p.stash_bytes() == o["stash_bytes"] and p.report["timeline"] == o["timeline"], st
        assert p.report["recompute_flops"] == o["recompute_flops"], st
    e = X.EchoPlan(m, (x,)).stash_bytes()
    b = X.EchoPlan(m, (x,), strategy="baseline").stash_bytes()
    assert e <= b
    _, saved = X.baseline_saved_bytes(m, x)
    assert saved == b


class _TanhGateMLP(nn.Module):
    """x <- tanh(W x) * sigmoid(G x) + x: tanh / sigmoid / mul / add maps between FCs."""

    def __init__(self, d=32, depth=3):
        super().__init__()
        self.fc = nn.ModuleList([nn.Linear(d, d) for _ in range(depth)])
        self.g = nn.ModuleList([nn.Linear(d, d) for _ in range(depth)])

    def forward(self, x):
        for f, g in zip(self.fc, self.g):
            x = torch.tanh(f(x)) * torch.sigmoid(g(x)) + x
        return x.sum()


class _GeluSiluMLP(nn.Module):
    """x <- x + W2 gelu(W1 x) * 0.5, then silu taps, F.gelu and a division by a constant."""

    def __init__(self, d=32, depth=2):
        super().__init__()
        self.w1 = nn.ModuleList([nn.Linear(d, 2 * d) for _ in range(depth)])
        self.w2 = nn.ModuleList([nn.Linear(2 * d, d) for _ in range(depth)])
        self.act = nn.GELU()
        self.tap = nn.SiLU()

    def forward(self, x):
        for a, b in zip(self.w1, self.w2):
            x = x + b(self.act(a(x))) * 0.5
        return (self.tap(x) / 4.0).sum() + torch.nn.functional.gelu(2.0 * x).sum()


class _PreLNBlock(nn.Module):
    """Transformer-style MLP blocks x <- x + W2 gelu(W1 LN(x)), a final F.layer_norm (no affine) and a
    linear head."""

    def __init__(self, d=32, depth=2):
        super().__init__()
        self.ln = nn.ModuleList([nn.LayerNorm(d) for _ in range(depth)])
        self.w1 = nn.ModuleList([nn.Linear(d, 4 * d) for _ in range(depth)])
        self.w2 = nn.ModuleList([nn.Linear(4 * d, d) for _ in range(depth)])
        self.head = nn.Linear(d, d)
        self.d = d

    def forward(self, x):
        for n, a, b in zip(self.ln, self.w1, self.w2):
            x = x + b(torch.nn.functional.gelu(a(n(x))))
        return self.head(torch.nn.functional.layer_norm(x, (self.d,))).sum()


@pytest.mark.parametrize("make,shape", [(lambda: ReluTaps(16, 3), (4, 16)), (lambda: ResMLP(16, 3), (4, 16)),
                                        (lambda: ResConvNet(4, 2), (2, 3, 8, 8)), (lambda: _TanhGateMLP(32, 3), (4, 32)),
                                        (lambda: _GeluSiluMLP(32, 2), (4, 32)), (lambda: _PreLNBlock(32, 2), (6, 32))],
                         ids=["relutaps", "resmlp", "resconv", "tanhgate", "gelusilu", "preln"])
def test_echo_module_plan_application_on_host(make, shape):
    """The saved-tensor-hook machinery of EchoModule on host tensors, for plans without 1-bit edges (the
    1-bit pack is a libecho kernel; the GPU test covers it): loss and every parameter gradient bitwise
    those of the unmodified model, the bytes the hooks keep == the estimator's Echo stash bytes, and the
    unmodified model's autograd keeps exactly the Baseline bytes."""
    from paper_1805_08899_b200 import fx_pass as X
    torch.manual_seed(0)
    m = make().double()
    x = torch.randn(*shape, dtype=torch.float64)
    ref, base_bytes = X.baseline_saved_bytes(m, x)
    ref.backward()
    g_ref = [p.grad.clone() for p in m.parameters()]
    m.zero_grad(set_to_none=True)
    em = X.EchoModule(m, (x,))
    assert "bit" not in set(em.plan.decision.values())
    assert base_bytes == X.EchoPlan(m, (x,), strategy="baseline").stash_bytes()
    loss = em(x)
    assert em.kept_bytes() == em.plan.stash_bytes() <= base_bytes
    loss.backward()
    assert torch.equal(loss.detach(), ref.detach())
    for p, g in zip(m.parameters(), g_ref):
        assert torch.equal(p.grad, g)

